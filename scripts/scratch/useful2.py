import sys, numpy as np
sys.path.insert(0, "/root/repo")
import synth, oracle
sc = synth.make_scene(3)
for vi in (0, 500, 900):
    cam = sc.cameras[vi]
    p = oracle.project(sc.field, cam)
    vis = np.nonzero(p["n_tiles"] > 0)[0]
    order = vis[np.lexsort((vis, p["depth_bits"][vis]))]
    rank = np.full(sc.field.n, -1, np.int64); rank[order] = np.arange(len(order))
    Nv = len(order)
    bs = oracle.bin_sort_batch([p], np.asarray(cam).reshape(1))
    gx, gy = oracle.grid(cam)
    rv = bs["ranges"][:gx * gy]; vals = bs["vals"]
    o = oracle.composite_tiled(p, vals, rv, cam)
    off, idx = oracle.composite_trace(p, vals, rv, cam)
    W = H = 800
    tf = o["t_final"].reshape(-1)
    sat = np.zeros(gx * gy, np.int64)  # depth-order index after which the tile is done (Nv = never)
    key_ranks = []
    for t in range(gx * gy):
        a, b = int(rv[t][0]), int(rv[t][1])
        if a == b: sat[t] = -1; key_ranks.append(np.zeros(0, np.int64)); continue
        kr = rank[vals[a:b]]; key_ranks.append(kr)
        ty, tx = divmod(t, gx)
        need = -1
        for yy in range(ty * 16, min(ty * 16 + 16, H)):
            for xx in range(tx * 16, min(tx * 16 + 16, W)):
                pi = yy * W + xx
                if tf[pi] >= 0.01: need = Nv; break
                bl = idx[off[pi]:off[pi + 1]]
                if len(bl): need = max(need, int(rank[int(bl[-1])]))
            if need == Nv: break
        sat[t] = need
    K = sum(len(k) for k in key_ranks)
    res = []
    for bounds in ([0.25], [0.35], [0.5], [0.2, 0.4, 0.7], [0.15, 0.3, 0.5, 0.75]):
        bnd = [int(f * Nv) for f in bounds] + [Nv]
        emitted = 0
        for t, kr in enumerate(key_ranks):
            if len(kr) == 0: continue
            prev = 0
            for bb in bnd:
                emitted += int(((kr >= prev) & (kr < bb)).sum())
                if sat[t] < bb: break   # done after this segment
                prev = bb
        res.append(f"{bounds}: {emitted / K:.3f}")
    print(f"view {vi}: K {K} Nv {Nv} ->", "; ".join(res), flush=True)
