// Example client of the C++ drop-in facade: the reference user's code with
// only the include changed.  Build:
//   g++ -O2 -std=c++17 -Iinclude examples/detect_loops.cpp
//       -Lpaper_2105_13168_b200/lib -ldifftopo_b200 -Wl,-rpath,$PWD/paper_2105_13168_b200/lib -o detect_loops
//   ./detect_loops torus:32:16:2:0.5 300
#include <cstdio>
#include <cstdlib>

#include "difftopo_b200.hpp"

int main(int argc, char** argv) {
  const std::string spec = argc > 1 ? argv[1] : "icosphere:3:2.0";
  difftopo::DiffusionConfig cfg;
  cfg.max_steps = argc > 2 ? std::atol(argv[2]) : 200000;
  try {
    auto mesh = spec.find('.') != std::string::npos && spec.find(':') == std::string::npos
                    ? difftopo::load_mesh(spec)
                    : difftopo::TriangleMesh::generate(spec);
    auto summary = difftopo::topology_summary(mesh);
    auto op = difftopo::assemble_laplacian(mesh);
    auto res = difftopo::run_initial_pass_partial(mesh, op, 0, cfg);
    std::printf("{\"V\":%u,\"genus\":%ld,\"status\":%d,\"steps\":%ld,\"events\":%zu,\"handle_estimates\":%ld}\n",
                summary.vertex_count, summary.genus, res.status, res.steps, res.events.size(),
                res.handle_estimate_count());
    for (const auto& ev : res.events) std::printf("  %s step=%ld layers=%zu\n", difftopo::to_string(ev.kind), ev.step, ev.layers.size());
    auto reeb = difftopo::build_reeb(res);
    std::printf("reeb: %zu nodes %zu arcs cycle_rank %ld\n", reeb.nodes.size(), reeb.edges.size(), reeb.cycle_rank());
    return res.status == DTB_OK ? 0 : 2;
  } catch (const difftopo::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
