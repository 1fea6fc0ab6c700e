import sys, numpy as np
sys.path.insert(0, "/root/repo")
import synth, oracle
sc = synth.make_scene(3)
for vi in (0, 500):
    cam = sc.cameras[vi]
    p = oracle.project(sc.field, cam)
    bs = oracle.bin_sort_batch([p], np.asarray(cam).reshape(1))
    gx, gy = oracle.grid(cam)
    rv = bs["ranges"][:gx * gy]
    vals = bs["vals"]
    o = oracle.composite_tiled(p, vals, rv, cam)
    off, idx = oracle.composite_trace(p, vals, rv, cam)
    W, H = 800, 800
    tf = o["t_final"].reshape(-1)
    total = useful = 0
    for ty in range(gy):
        for tx in range(gx):
            a, b = int(rv[ty * gx + tx][0]), int(rv[ty * gx + tx][1])
            L = b - a
            if L == 0: continue
            pos = {int(g): i for i, g in enumerate(vals[a:b])}
            need = 0
            for yy in range(ty * 16, min(ty * 16 + 16, H)):
                for xx in range(tx * 16, min(tx * 16 + 16, W)):
                    pi = yy * W + xx
                    if tf[pi] >= 0.01: need = L; break
                    bl = idx[off[pi]:off[pi + 1]]
                    need = max(need, pos[int(bl[-1])] + 1 if len(bl) else 0)
                if need == L: break
            total += L; useful += need
    print(f"view {vi}: keys {total}, useful prefix {useful} ({useful/total:.3f})")
