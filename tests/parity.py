"""Comparison of the device engine's outputs with the reference's (test-only)."""
import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    x = np.asarray(x, np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def entry_hash_sum(layer, verts, vals):
    """Sum of splitmix64(splitmix64((layer << 40) ^ v) ^ bits(x)) mod 2^64."""
    v = np.asarray(verts, np.uint64)
    bits = np.asarray(vals, np.float64).view(np.uint64)
    h = splitmix64(splitmix64((np.uint64(layer) << np.uint64(40)) ^ v) ^ bits)
    with np.errstate(over="ignore"):
        return int(np.sum(h, dtype=np.uint64))


def compare_events(mine, ref_events, vanish_tol=1e-9, check_covered=True):
    """Event logs must agree exactly in kind, step, layers, produced, loops and
    covered sets; split/merge positions bit for bit (host-exact sums); vanish
    positions within vanish_tol (device fixed-point band means)."""
    assert len(mine) == len(ref_events), (len(mine), len(ref_events))
    for i, (a, b) in enumerate(zip(mine, ref_events)):
        where = f"event {i} ({b['kind']} @ {b['step']})"
        assert a.kind == b["kind"], where
        assert a.step == b["step"], where
        assert a.layers == b["layers"], where
        assert a.produced == b["produced"], where
        if a.kind == "vanish":
            assert np.allclose(a.position, b["position"], rtol=0, atol=vanish_tol), (where, a.position, b["position"])
        elif a.kind != "seed":
            assert tuple(a.position) == tuple(b["position"]), (where, a.position, b["position"])
        if check_covered and a.covered is not None:
            assert np.array_equal(a.covered, np.asarray(b["covered"], np.uint32)), where
        assert len(a.estimates) == len(b["estimates"]), where
        for ea, eb in zip(a.estimates, b["estimates"]):
            assert ea.layer == eb["layer"], where
            assert ea.length == eb["length"], where
            assert len(ea.points) == len(eb["points"]), where
            for pa, pb in zip(ea.points, eb["points"]):
                assert (pa.edge, pa.t, pa.face) == (pb[0], pb[1], pb[2]), where
                assert tuple(pa.position) == tuple(pb[3]), where
            assert len(ea.snapshot[0]) == eb["snapshot_n"], where
            assert entry_hash_sum(ea.layer, *ea.snapshot) == int(eb["snapshot_hash"]), where


def compare_tracks(mine, ref_tracks, trail_tol=None):
    assert len(mine) == len(ref_tracks)
    exact = total = 0
    for a, b in zip(mine, ref_tracks):
        assert (a["layer"], a["created"], a["consumed"]) == (b["layer"], b["created"], b["consumed"])
        assert len(a["trail"]) == len(b["trail"]), (a["layer"], len(a["trail"]), len(b["trail"]))
        if len(b["trail"]):
            rb = np.asarray(b["trail"])
            exact += int(np.sum(np.all(a["trail"] == rb, axis=1)))
            total += len(rb)
            if trail_tol is not None:
                assert np.max(np.abs(a["trail"] - rb)) <= trail_tol
    return exact, total
