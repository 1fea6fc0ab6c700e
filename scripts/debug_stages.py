"""Stage-by-stage GPU vs oracle comparison (debug aid; prints, never asserts)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2602_15355_b200 import Context, gsr  # noqa: E402
from tests.gpu_utils import oracle_batch, to_dev  # noqa: E402


def cmp(name, a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        print(f"  {name}: SHAPE {a.shape} vs {b.shape}")
        return
    bad = np.nonzero(a.reshape(-1) != b.reshape(-1))[0]
    print(f"  {name}: {len(bad)} / {a.size} mismatches" + (f" first at {bad[:5]} gpu={a.reshape(-1)[bad[:5]]} orc={b.reshape(-1)[bad[:5]]}" if len(bad) else ""))


def run(field, cams, label):
    print(f"== {label}: n={field.n} V={len(cams)} {int(cams[0]['width'])}x{int(cams[0]['height'])}")
    ctx = Context(0)
    G = to_dev(field)
    V, n = len(cams), field.n
    W, H = int(cams[0]["width"]), int(cams[0]["height"])
    T = V * ((W + 15) // 16) * ((H + 15) // 16)
    o = oracle_batch(field, cams, images=True)
    rec = torch.zeros((V, n, 12), device="cuda")
    binr = torch.zeros(10 * V * n, dtype=torch.int32, device="cuda")
    gsr.gsr_project(ctx, G, cams, rec, binr)
    torch.cuda.synchronize()
    b = binr.cpu().numpy().view(np.uint32)[8 * V * n:].reshape(2, V, n)  # depth, n_tiles planes
    for v, p in enumerate(o["projs"]):
        if v < 2 or v == V - 1:
            cmp(f"view{v} n_tiles", b[1, v], p["n_tiles"])
            cmp(f"view{v} depth", b[0, v], p["depth_bits"])
    K = len(o["keys"])
    print("  oracle K", K)
    vals = torch.full((K + 16,), -1, dtype=torch.int32, device="cuda")
    keys = torch.full((K + 16,), -1, dtype=torch.int64, device="cuda")
    ku = torch.full((K + 16,), -1, dtype=torch.int64, device="cuda")
    vu = torch.full((K + 16,), -1, dtype=torch.int32, device="cuda")
    ranges = torch.full((T, 2), -1, dtype=torch.int32, device="cuda")
    Kg = gsr.gsr_bin_sort(ctx, binr, n, cams, vals, K + 16, ranges, keys=keys, keys_unsorted=ku, vals_unsorted=vu)
    torch.cuda.synchronize()
    print("  gpu K", Kg)
    cmp("keys_unsorted", ku.cpu().numpy().view(np.uint64)[:K], o["keys_unsorted"])
    cmp("vals_unsorted", vu.cpu().numpy().view(np.uint32)[:K], o["vals_unsorted"])
    gk = keys.cpu().numpy().view(np.uint64)[:K]
    gv = vals.cpu().numpy().view(np.uint32)[:K]
    cmp("keys", gk, o["keys"])
    cmp("vals", gv, o["vals"])
    cmp("ranges", ranges.cpu().numpy().view(np.uint32), o["ranges"])
    cmp("tile of keys", gk >> np.uint64(32), o["keys"] >> np.uint64(32))
    print("  gpu keys sorted?", bool(np.all(gk[1:] >= gk[:-1])), "vals<n", bool(np.all(gv < n)))
    part = torch.zeros(T, device="cuda")
    rgbu = torch.zeros((V, H, W, 4), device="cuda")
    nc = torch.zeros((V, H, W), dtype=torch.int32, device="cuda")
    # composite with the ORACLE's sorted values, to isolate K6
    ov = torch.from_numpy(o["vals"].view(np.int32).copy()).cuda()
    orng = torch.from_numpy(o["ranges"].view(np.int32).copy()).cuda()
    gsr.gsr_composite(ctx, rec, n, ov, orng, cams, part, rgbu=rgbu, n_contrib=nc)
    torch.cuda.synchronize()
    d = np.abs(rgbu.cpu().numpy() - o["rgbu"])
    print("  composite(oracle lists): max |d|", d.max(), "n_contrib mismatches",
          int((nc.cpu().numpy().view(np.uint32) != o["n_contrib"]).sum()))


if __name__ == "__main__" and "--sort" not in sys.argv:
    sc = synth.make_scene(1, n_override=2000, views=4)
    run(sc.field, sc.cameras, "smoke-like")
    sc = synth.make_scene(1)
    run(sc.field, sc.cameras[:2], "c1 2 views")
    run(sc.field, sc.cameras, "c1 16 views")


def sort_check():
    ctx = Context(0)
    rng = np.random.default_rng(0)
    for n in (100, 3072, 3073, 10000, 50000):
        for bits in ((0, 8), (0, 16), (0, 36), (8, 20)):
            k = rng.integers(0, 2 ** 36, n, dtype=np.int64).astype(np.uint64)
            v = np.arange(n, dtype=np.uint32)
            kin = torch.from_numpy(k.view(np.int64)).cuda()
            vin = torch.from_numpy(v.view(np.int32)).cuda()
            ko = torch.empty_like(kin)
            vo = torch.empty_like(vin)
            gsr.gsr_sort_pairs_u64(ctx, kin, vin, ko, vo, bits[0], bits[1])
            torch.cuda.synchronize()
            d = (k >> np.uint64(bits[0])) & np.uint64((1 << (bits[1] - bits[0])) - 1)
            o = np.argsort(d, kind="stable")
            gv = vo.cpu().numpy().view(np.uint32)
            print(f"sort n={n} bits={bits}: val mismatches {(gv != v[o]).sum()}  perm? {len(np.unique(gv)) == n}")


if "--sort" in sys.argv:
    sort_check()
