// Example: a batch of independent meshes (BASELINE configs[4]) through the
// C++ facade's run_initial_pass_batch, several passes at once on one GPU.
//   g++ -O2 -std=c++17 -Iinclude examples/batch_passes.cpp
//       -Lpaper_2105_13168_b200/lib -ldifftopo_b200 -Wl,-rpath,$PWD/paper_2105_13168_b200/lib -o batch_passes
//   ./batch_passes 16 300
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "difftopo_b200.hpp"

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 16;
  difftopo::DiffusionConfig cfg;
  cfg.max_steps = argc > 2 ? std::atol(argv[2]) : 3000;
  try {
    difftopo::init_work_queues(32);  // opt-in, before any CUDA use: 16 passes at once need 16+ hardware queues
    std::vector<difftopo::TriangleMesh> meshes;
    std::vector<difftopo::LaplacianOperator> ops;
    for (int i = 0; i < n; ++i) meshes.push_back(difftopo::TriangleMesh::generate("genus:" + std::to_string(1 + i % 32) + ":3"));
    for (const auto& m : meshes) ops.push_back(difftopo::assemble_laplacian(m));
    std::vector<const difftopo::TriangleMesh*> mp;
    std::vector<const difftopo::LaplacianOperator*> op;
    for (int i = 0; i < n; ++i) {
      mp.push_back(&meshes[i]);
      op.push_back(&ops[i]);
    }
    auto res = difftopo::run_initial_pass_batch(mp, op, std::vector<difftopo::Index>(n, 0), cfg);
    for (int i = 0; i < n; ++i)
      std::printf("{\"item\":%d,\"status\":%d,\"steps\":%ld,\"events\":%zu}\n", i, res[i].status, res[i].steps,
                  res[i].events.size());
    return 0;
  } catch (const difftopo::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
