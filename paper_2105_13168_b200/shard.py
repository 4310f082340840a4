"""Sharding of independent meshes / seeds across ranks (one process per GPU).

The initial pass of one mesh is a single global front: every step ends in a
grid-wide barrier, so a pass never spans GPUs.  What shards is the batch --
independent meshes or seed vertices (BASELINE configs[4]: 64 synthetic
genus-1..32 meshes on 1/2/4/8 B200).  Each rank runs its slice with no
data-path collective; only the per-item summaries are gathered at the end
(`torch.distributed.gather_object`, NCCL or gloo)."""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence


def shard(items: Sequence, rank: int, world: int) -> List:
    """Round-robin slice of `items` for `rank` (balanced for sorted sizes)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(items[rank::world])


def batch_specs(n: int = 64, max_genus: int = 32, resolution: int = 3) -> List[str]:
    """configs[4]: n synthetic meshes of genus 1..max_genus (generate_genus_g)."""
    return [f"genus:{1 + (i % max_genus)}:{resolution}" for i in range(n)]


def run_item(spec: str, max_steps: int, seed: int = 0) -> dict:
    """One independent initial pass on this rank's GPU; returns a summary."""
    from . import TriangleMesh, assemble_laplacian, default_config, run_initial_pass

    mesh = TriangleMesh.generate(spec)
    op = assemble_laplacian(mesh)
    res = run_initial_pass(mesh, op, seed, default_config(max_steps=max_steps))
    tm = res.timing()
    info = mesh.info()
    return {"spec": spec, "V": info["V"], "genus": info["genus"], "status": res.status, "steps": res.steps,
            "events": res.n_events, "handle_estimates": res.handle_estimate_count, "t_pass": tm["t_pass_device"],
            "field_hash": res.field_hash()}


def run_batch(specs: Sequence[str], max_steps: int, seed: int = 0, concurrency: int = 0,
              arrays: Optional[dict] = None) -> List[dict]:
    """This rank's items as one native batch (dtb_run_initial_pass_batch):
    meshes and operators are built first, then the passes run several at a
    time on disjoint SM shares; each summary equals run_item's.  `arrays`
    (spec -> (vertices, faces)) supplies host arrays instead of generating."""
    from . import TriangleMesh, assemble_laplacian, default_config, run_initial_pass_batch

    meshes = [TriangleMesh.from_arrays(*arrays[s]) if arrays else TriangleMesh.generate(s) for s in specs]
    ops = [assemble_laplacian(m) for m in meshes]
    res = run_initial_pass_batch(meshes, ops, [seed] * len(specs), default_config(max_steps=max_steps),
                                 concurrency=concurrency)
    out = []
    for spec, mesh, r in zip(specs, meshes, res):
        info = mesh.info()
        out.append({"spec": spec, "V": info["V"], "genus": info["genus"], "status": r.status, "steps": r.steps,
                    "events": r.n_events, "handle_estimates": r.handle_estimate_count,
                    "t_pass": r.timing()["t_pass_device"], "field_hash": r.field_hash()})
    return out


def run_sharded_batch(items: Sequence, rank: int, world: int, max_steps: int, dist=None,
                      concurrency: int = 0, arrays: Optional[dict] = None) -> List[dict]:
    """run_sharded with this rank's slice run as one concurrent batch."""
    mine = shard(items, rank, world)
    res = run_batch(mine, max_steps, concurrency=concurrency, arrays=arrays)
    out = [dict(r, index=rank + world * k) for k, r in enumerate(res)]
    return _gather(out, rank, world, dist)


def run_sharded(items: Sequence, rank: int, world: int, worker: Callable[[object], dict], dist=None) -> List[dict]:
    """Runs `worker` on this rank's slice; rank 0 returns every item's result
    in the original order (other ranks return their own slice)."""
    mine = shard(items, rank, world)
    out = [dict(worker(it), index=rank + world * k) for k, it in enumerate(mine)]
    return _gather(out, rank, world, dist)


def _gather(out: List[dict], rank: int, world: int, dist) -> List[dict]:
    if dist is None or world == 1:
        return out
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(out, gathered, dst=0)
    if rank != 0:
        return out
    merged = [r for part in gathered for r in part]
    merged.sort(key=lambda r: r["index"])
    return merged
