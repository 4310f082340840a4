#!/usr/bin/env python
"""Benchmark of the diffusion-front initial pass (arXiv 2105.13168 handle/tunnel
detector) on B200.

Metric (BASELINE.json): "end-to-end handle/tunnel detection ms per mesh;
diffusion Mvert-steps/s".  A bench *step* is one full invocation of the hot
path -- run_initial_pass (reference diffusion.hpp:861) with the default
DiffusionConfig and max_steps = --pass-steps -- on configs[1], the genus-8
subdivided multi-handle surface (generate_genus_g(8, 45): 988,186 vertices).
On that mesh the reference's initial pass does not terminate, so every pass
(reference and ours) stops with MaxStepsExceeded after exactly --pass-steps
explicit-Euler steps, each followed by the full front check (CCL, collision
detection, events).  ``value`` = mesh vertices x diffusion steps / second
(Mvert-steps/s, whole job over all ranks); ``ms_per_step`` = ms per pass.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Under torchrun each rank runs an independent copy of the workload (seed
vertex = rank): the path shards by mesh/seed with no data-path collective
(weak scaling); ranks meet only at the timing barriers.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "end-to-end handle/tunnel detection ms per mesh; diffusion Mvert-steps/s"
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "difftopo_ref")
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")

# Algorithmic bytes per unit of work of the persistent step kernel
# (DESIGN.md "Roofline"): a frontier vertex reads its column (1 + 2 x 10 B),
# its stiffness row (8 B offsets + 7 x 12 B), its mass (8 B) and its 7
# neighbours' columns (7 x 21 B), and writes its new column (21 B) -> 288 B
# (round 1 staged the column in scratch and committed it: 330 B).  A band vertex of the
# check reads its column (21 B), its front-connectivity row (8 + 12 x 4 B),
# the 6 higher-numbered neighbours' columns (6 x 21 B), union-find parents
# (2 x 8 B) and its fixed-point position (24 B) -> 243 B; the band scan
# reads one flag byte per mesh vertex.
BYTES_PER_FRONTIER_VERTEX = 288
BYTES_PER_BAND_VERTEX = 243
BYTES_PER_MESH_VERTEX_SCAN = 1


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--mesh", default="genus:8:45")
    p.add_argument("--pass-steps", type=int, default=3000)
    p.add_argument("--no-e2e", action="store_true")
    return p.parse_args()


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world == 1:
        return rank, world, local, None
    import torch
    import torch.distributed as tdist
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(local)
    tdist.init_process_group(backend=backend)
    return rank, world, local, tdist


def barrier(tdist):
    if tdist is not None:
        tdist.barrier()


def max_over_ranks(tdist, x):
    if tdist is None:
        return x
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 9:
                continue
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def l2_flush(buf):
    if buf is not None:
        buf.add_(1.0)


def cpu_reference_sample(spec, steps):
    """The reference's own initial pass (oracle/_ref, compiled from the
    unmodified headers) timed on this host for a bounded number of steps."""
    if not os.path.exists(REF_BIN):
        return None
    out = subprocess.run([REF_BIN, "time", spec, f"max_steps={steps}"], check=True, capture_output=True, text=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def measured_traffic(args):
    """DRAM bytes per k_engine launch from the committed ncu --set full capture
    (profiles/traffic_k_engine.json), when it was taken on this workload."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic_k_engine.json")
    if args.mesh != "genus:8:45" or args.pass_steps != 3000 or not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh)["dram_bytes_per_launch"]  # bytes per launch, like alg_bytes_per_launch


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload_config(args, V, world):
    """The config both arms print (identical dicts, so the driver can pair them)."""
    parts = args.mesh.split(":")
    genus = int(parts[1]) if parts[0] == "genus" and len(parts) > 1 else None
    return {"workload": f"run_initial_pass on {args.mesh} (configs[1]: genus-8 subdivided multi-handle surface), "
                        f"max_steps={args.pass_steps}; e2e and the reference arm also build the mesh and "
                        f"assemble the Laplacian from host arrays",
            "mesh": args.mesh, "vertices": V, "genus": genus, "pass_steps": args.pass_steps,
            "seed_vertex": "rank % V (0 at N=1)", "parallelism": f"replicas x{world}",
            "l2": "GPU arm: 256 MiB buffer rewritten before every timed pass"}


def reference_concurrency(k):
    """Independent reference passes run at once: one per host core the process
    may use, bounded by memory (~1.5 GB per 1M-vertex pass)."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        with open("/proc/meminfo") as fh:
            avail = next(int(l.split()[1]) for l in fh if l.startswith("MemAvailable")) * 1024
        by_mem = max(1, int(avail // (3 << 29)))
    except (OSError, StopIteration):
        by_mem = cores
    return max(1, min(k, cores, by_mem))


def reference_wave(spec, steps, n):
    """n concurrent single-threaded reference passes (separate processes);
    returns their JSON reports."""
    procs = [subprocess.Popen([REF_BIN, "time", spec, f"max_steps={steps}"], stdout=subprocess.PIPE,
                              stderr=subprocess.DEVNULL, text=True) for _ in range(n)]
    out = []
    for p in procs:
        so, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"reference pass exited {p.returncode}")
        out.append(json.loads(so.strip().splitlines()[-1]))
    return out


def run_reference_arm(args, rank, world, tdist):
    """The reference's own CPU implementation (oracle/_ref, compiled from the
    unmodified headers) on the same workload, end to end: TriangleMesh
    construction + assemble_laplacian + run_initial_pass for --pass-steps
    steps -- the same stages the b200 arm's e2e times through the C ABI.
    The reference pass is single-threaded, so the arm uses the host's cores
    the way the b200 arm uses GPUs: independent passes side by side, as many
    at once as there are cores (and memory).  A step is one pass; the K
    timed passes run in balanced waves of at most that width, each pass
    timed by the reference's own setup + pass clocks, and the host's
    throughput is width passes per mean pass time."""
    if rank != 0:
        return
    if not os.path.exists(REF_BIN):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/difftopo_ref not built"}))
        return
    S = args.pass_steps
    width = reference_concurrency(args.steps)
    if args.warmup > 0:  # pages the binary and the allocator in; nothing carries over between processes
        reference_wave(args.mesh, S, min(args.warmup, width))
    V, per_pass, setup = None, [], []
    waves = -(-args.steps // width)
    sizes = [args.steps // waves + (1 if i < args.steps % waves else 0) for i in range(waves)]  # balanced waves
    for n in sizes:
        reps = reference_wave(args.mesh, S, n)
        V = reps[0]["V"]
        per_pass += [r["seconds"] for r in reps]
        setup += [r["setup_seconds"] for r in reps]
    # Throughput of `width` cores each running passes back to back: every
    # pass on its own clock (setup + pass, measured while its wave shares
    # the host), amortised over the cores.
    total = (sum(per_pass) + sum(setup)) / width
    value = V * S * args.steps / total / 1e6
    line = {
        "metric": METRIC, "value": value, "unit": "Mvert-steps/s", "impl": "reference", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, V, world),
        "ms_per_mesh": 1e3 * total / args.steps,
        "ms_per_pass_single": 1e3 * statistics.median(per_pass),
        "ms_setup_single": 1e3 * statistics.median(setup),
        "cpu_baseline": {"value": value, "unit": "Mvert-steps/s", "cores": width, "kind": "reference",
                         "sample": f"{args.steps} full {S}-step initial passes from vertex 0 on {args.mesh} "
                                   f"(V={V}), each with its mesh and operator setup; single-threaded reference "
                                   f"passes, {width} at a time on {width} host cores"},
        "e2e": {"value": value, "unit": "Mvert-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    args = parse()
    rank, world, local, tdist = dist_setup()
    if args.impl == "reference":
        run_reference_arm(args, rank, world, tdist)
        if tdist is not None:
            tdist.destroy_process_group()
        return

    import torch
    import paper_2105_13168_b200 as dt

    torch.cuda.set_device(local)
    dt.device_info()
    mesh = dt.TriangleMesh.generate(args.mesh)
    info = mesh.info()
    V = info["V"]
    op = dt.assemble_laplacian(mesh)
    cfg = dt.default_config(max_steps=args.pass_steps)
    seed = rank % V
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    def one_pass():
        res = dt.run_initial_pass(mesh, op, seed, cfg)
        return res

    for _ in range(args.warmup):
        one_pass()
    torch.cuda.synchronize()

    # ---- device-resident timed region
    pass_times, kern_times, work = [], [], []
    launches0 = dt.launch_count()
    with ClockSampler(local) as clocks:
        barrier(tdist)
        torch.cuda.synchronize()
        for _ in range(args.steps):
            l2_flush(flush)
            torch.cuda.synchronize()
            res = one_pass()
            tm = res.timing()
            pass_times.append(tm["t_pass_device"])
            kern_times.append((tm["t_kernel"], tm["launches"]))
            work.append(tm)
            status, steps_done = res.status, res.steps
            del res
        torch.cuda.synchronize()
        barrier(tdist)
    gpu_launches = dt.launch_count() - launches0
    total = max_over_ranks(tdist, sum(pass_times))
    value = world * V * args.pass_steps * args.steps / total / 1e6

    # ---- roofline of the dominant kernel (the persistent step kernel)
    k_time = sum(k for k, _ in kern_times)
    k_launches = sum(n for _, n in kern_times)
    sum_region = sum(w["sum_region"] for w in work)
    sum_band = sum(w["sum_interest"] for w in work)
    alg_bytes = (BYTES_PER_FRONTIER_VERTEX * sum_region + BYTES_PER_BAND_VERTEX * sum_band +
                 BYTES_PER_MESH_VERTEX_SCAN * V * args.pass_steps * args.steps)
    achieved = alg_bytes / k_time / 1e9
    peak, peak_kind = peaks()

    # ---- the full-mesh operator sweep (what a dense formulation reads every step)
    sw = op.sweep_bench(10)
    dense = {"kernel": "k_spmv_ell (y = M^-1 S x over all V rows, padded 8-entry rows)",
             "us_per_sweep": 1e6 * sw["seconds"], "achieved": sw["gbs"], "peak": peak, "unit": "GB/s",
             "frac": sw["gbs"] / peak, "alg_bytes_per_sweep": sw["bytes"],
             "frontier_us_per_step": 1e6 * total / args.steps / args.pass_steps,
             "note": "each sweep after a 256 MiB L2-evicting read; a dense step would pay at least this "
                     "every step, the frontier step touches ~0.6 % of V"}

    # ---- end-to-end through the C ABI from host buffers
    e2e = None
    if not args.no_e2e:
        verts, faces = mesh.vertices(), mesh.faces()
        vpin = torch.from_numpy(verts).pin_memory().numpy()
        fpin = torch.from_numpy(faces.astype(np.int32)).pin_memory().numpy().view(np.uint32)
        e2e_times, h2d, d2h = [], 0, 0
        for i in range(args.warmup + args.steps):
            l2_flush(flush)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m = dt.TriangleMesh.from_arrays(vpin, fpin)
            o = dt.assemble_laplacian(m)
            r = dt.run_initial_pass(m, o, seed, cfg)
            evs = r.events()
            trs = r.tracks()
            t1 = time.perf_counter()
            if i >= args.warmup:
                e2e_times.append(t1 - t0)
                h2d = m.upload_bytes()  # positions, faces and the host-built mesh index
                d2h = (sum(32 + (e.covered.nbytes if e.covered is not None else 0) +
                           sum(len(x.points) * 40 + x.snapshot[0].nbytes + x.snapshot[1].nbytes for x in e.estimates)
                           for e in evs) + sum(t["trail"].nbytes + 24 for t in trs))
            del r, o, m
        e2e_total = max_over_ranks(tdist, sum(e2e_times))
        e2e = {"value": world * V * args.pass_steps * args.steps / e2e_total / 1e6, "unit": "Mvert-steps/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_mesh": 1e3 * e2e_total / args.steps,
               "includes": "H2D of the vertex/face arrays, device mesh validation/orientation/indexing, device "
                           "Laplacian assembly, initial pass, D2H of events/estimates/covered sets/trails"}

    line = {
        "metric": METRIC, "value": value, "unit": "Mvert-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, V, world),
        "pass_status": status, "steps_per_pass": steps_done, "genus_measured": info["genus"],
        "ms_per_mesh": 1e3 * total / args.steps,
        "gpu_launches": int(gpu_launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": measured_traffic(args), "traffic_unit": "DRAM bytes per launch (ncu)",
                     "peak_kind": peak_kind,
                     "limiter": "latency: per step a chain of dependent L2 round trips (frontier list, columns, "
                                "neighbour columns, one-ring claims) and FP64 update arithmetic, then one grid "
                                "barrier; the working set stays in L2 (traffic vs alg_bytes_per_launch)",
                     "kernel": "k_engine<0> (persistent step kernel)",
                     "kernel_seconds": k_time, "kernel_launches": k_launches,
                     "alg_bytes_per_launch": alg_bytes / max(1, k_launches),
                     "avg_frontier_vertices_per_step": sum_region / (args.pass_steps * args.steps),
                     "avg_band_vertices_per_step": sum_band / (args.pass_steps * args.steps)},
        "clocks": clocks.summary(),
        "e2e": e2e,
        "dense_sweep": dense,
    }
    if rank == 0 and world == 1:
        S = args.pass_steps
        r = cpu_reference_sample(args.mesh, S)
        if r is not None:
            line["cpu_baseline"] = {"value": V * S / r["seconds"] / 1e6, "unit": "Mvert-steps/s", "cores": 1,
                                    "kind": "reference",
                                    "sample": f"first {S} initial-pass steps from vertex 0 on {args.mesh} "
                                              f"(V={V}), single-threaded reference ({r['seconds']:.2f} s)"}
    if rank == 0:
        print(json.dumps(line))
    if tdist is not None:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
