"""Work model of the blend (K6) at a BASELINE config, computed on the CPU from
the reference's own prepared splats and tile lists (oracle/_ref): per tile and
per 8x8 warp block, how many candidate steps the pixel-pair walk takes, how
far down its list a tile's last pixel terminates, and how the work spreads
over tiles. Design-study tool (not a test; not used by the product).

    python tools/blend_model.py [--n 1000000] [--seed 2] [--kernel poly1] [--mode OpacityAware]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle  # noqa: E402
from paper_2603_18707_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--seed", type=int, default=2)
ap.add_argument("--w", type=int, default=1920)
ap.add_argument("--h", type=int, default=1080)
ap.add_argument("--kernel", default="poly1")
ap.add_argument("--mode", default="OpacityAware")
ap.add_argument("--tiles", type=int, default=0, help="model only every k-th tile (0: all)")
a = ap.parse_args()

ref = oracle.Reference()
splats, deg = ref.synth_g(a.n, a.seed)
cam = ref.orbit_cameras(256, a.w, a.h)[0]
cfg = api.RasterConfig(kernel=api.fitted_kernel(a.kernel), culling_mode=getattr(api.CullingMode, a.mode),
                       sh_degree=deg).to_struct()
prep = ref.prepare(splats, cam, cfg)
off, idx, ctr = ref.tile_lists(splats, cam, cfg)
print("counters", ctr, file=sys.stderr)
row = np.full(a.n, -1, np.int64)
row[prep.index] = np.arange(len(prep.index))
k = cfg.kernel
coef = np.array([k.coeffs[j] for j in range(k.order + 1)])
eps, floor = cfg.epsilon, cfg.transmittance_floor
ts = 16
tx_n = (a.w + ts - 1) // ts
ty_n = (a.h + ts - 1) // ts
ly, lx = np.mgrid[0:16, 0:16]
stats = []
group_stats = []
quad_stats = []
step = a.tiles if a.tiles > 0 else 1
for t in range(0, tx_n * ty_n, step):
    lst = idx[off[t]:off[t + 1]]
    L = len(lst)
    if L == 0:
        continue
    r = row[lst]
    tx, ty = t % tx_n, t // tx_n
    gx = (tx * 16 + lx).ravel()
    gy = (ty * 16 + ly).ravel()
    inside = (gx < a.w) & (gy < a.h)
    m = prep.mean2d[r]
    cn = prep.conic[r]
    o = prep.opacity_eff[r]
    dx = (gx[None, :] + 0.5) - m[:, 0:1]
    dy = (gy[None, :] + 0.5) - m[:, 1:2]
    q = cn[:, 0:1] * dx * dx + 2.0 * cn[:, 1:2] * dx * dy + cn[:, 2:3] * dy * dy
    if k.kind == 0:
        kv = np.exp(-0.5 * q)
    else:
        kv = np.polyval(coef[::-1], q)
        kv = np.maximum(kv, 0.0) if k.kind == 1 else np.where(q < k.first_root, kv, 0.0)
    al = np.minimum(0.999, o[:, None] * kv)
    acc = al >= eps                                   # [L, 256]
    om = np.where(acc, 1.0 - al, 1.0)
    Tb = np.cumprod(np.vstack([np.ones((1, 256)), om[:-1]]), axis=0)  # T before entry k
    stop = acc & (Tb * (1.0 - al) < floor)
    has = stop.any(axis=0)
    term = np.where(has, stop.argmax(axis=0), L)      # list position of the stop (L: none)
    live = np.arange(L)[:, None] < term[None, :]      # entries a pixel still visits
    live_inc = np.arange(L)[:, None] <= np.minimum(term, L - 1)[None, :]
    cand = acc & live_inc & inside[None, :]           # per-pixel candidate steps (incl. the stop)
    # pixel pairs (2k, 2k+1) of each row: the walk's step set is the union
    c2 = cand.reshape(L, 16, 8, 2)
    pair_steps = (c2[..., 0] | c2[..., 1]).sum(axis=0)  # [16 rows, 8 pairs]
    c4 = cand.reshape(L, 16, 4, 4).any(axis=3)           # 1x4 quads: [L, 16 rows, 4 quads]
    q14 = c4.sum(axis=0)
    c22 = cand.reshape(L, 8, 2, 8, 2).any(axis=(2, 4))   # 2x2 quads: [L, 8, 8]
    q22 = c22.sum(axis=0)
    # 1x4: warp = 8 rows x 4 quads (half tile); SIMT max per warp
    w14 = [int(q14[h * 8:(h + 1) * 8].max()) for h in range(2)]
    w22 = [int(q22[(h >> 1) * 4:(h >> 1) * 4 + 4, (h & 1) * 4:(h & 1) * 4 + 4].max()) for h in range(4)]
    quad_stats.append((int(q14.sum()), sum(w14), int(q22.sum()), sum(w22)))
    # warp blocks: rows (w>>1)*8.., pairs (w&1)*4..
    ws = [pair_steps[(w >> 1) * 8:(w >> 1) * 8 + 8, (w & 1) * 4:(w & 1) * 4 + 4] for w in range(4)]
    # per group of 32 records: the warp's step count is the max over its lanes
    pc = (c2[..., 0] | c2[..., 1])                       # [L, 16, 8] pair candidates
    ng = (L + 31) // 32
    pcg = np.zeros((ng * 32, 16, 8), bool)
    pcg[:L] = pc
    per_g = pcg.reshape(ng, 32, 16, 8).sum(axis=1)       # [ng, 16, 8]
    gmax = sum(int(per_g[:, (w >> 1) * 8:(w >> 1) * 8 + 8, (w & 1) * 4:(w & 1) * 4 + 4].reshape(ng, -1).max(axis=1).sum())
               for w in range(4))
    gm2 = []
    for G in (64, 128):
        ngG = (L + G - 1) // G
        pcG = np.zeros((ngG * G, 16, 8), bool)
        pcG[:L] = pc
        perG = pcG.reshape(ngG, G, 16, 8).sum(axis=1)
        gm2.append(sum(int(perG[:, (w >> 1) * 8:(w >> 1) * 8 + 8, (w & 1) * 4:(w & 1) * 4 + 4].reshape(ngG, -1).max(axis=1).sum())
                       for w in range(4)))
    group_stats.append((gmax, gm2[0], gm2[1]))
    evals = np.where(inside, np.minimum(term + 1, L), 0).sum()
    blended = (acc & live & inside[None, :]).sum()
    last = int(np.where(inside, np.minimum(term + 1, L), 0).max())   # entries the tile needs
    tn = np.where(inside, np.minimum(term + 1, L), 0).reshape(16, 16)
    blast = [int(tn[(w >> 1) * 8:(w >> 1) * 8 + 8, (w & 1) * 8:(w & 1) * 8 + 8].max()) for w in range(4)]
    # records (before the block's last termination) whose {alpha >= eps} meets the block
    ab = acc.reshape(L, 16, 16)
    btouch = [int(ab[:blast[w], (w >> 1) * 8:(w >> 1) * 8 + 8, (w & 1) * 8:(w & 1) * 8 + 8].any(axis=(1, 2)).sum())
              for w in range(4)]
    stats.append((t, L, last, int(cand.sum()), int(pair_steps.sum()),
                  [int(x.max()) for x in ws], [int(x.sum()) for x in ws], int(evals), int(blended), blast, btouch))

L = np.array([s[1] for s in stats])
last = np.array([s[2] for s in stats])
cand = np.array([s[3] for s in stats])
psteps = np.array([s[4] for s in stats])
wmax = np.array([s[5] for s in stats])
wsum = np.array([s[6] for s in stats])
ev = np.array([s[7] for s in stats])
bl = np.array([s[8] for s in stats])
blast = np.array([s[9] for s in stats])
btouch = np.array([s[10] for s in stats])
print(f"per-block prefix (records a warp must scan) {blast.sum()} = {blast.sum() / (4 * last.sum()):.3f} x 4 x tile prefix; "
      f"records meeting the block {btouch.sum()} ({btouch.sum() / blast.sum():.3f} of scanned)")
print(f"tiles {len(stats)}  pairs {L.sum()}  evals {ev.sum()}  blended {bl.sum()}")
print(f"records staged (whole lists) {L.sum()}  needed (to the tile's last termination) {last.sum()} "
      f"({last.sum() / L.sum():.3f})")
print(f"per-pixel candidate steps {cand.sum()}  pair-walk steps {psteps.sum()} "
      f"(x{psteps.sum() * 2 / cand.sum():.3f} pixel slots per candidate)")
print(f"warp walk steps (max over lanes) {wmax.sum()}  lane-steps {wsum.sum()}  "
      f"SIMT efficiency {wsum.sum() / (32 * wmax.sum()):.3f}")
print(f"per tile: L mean {L.mean():.0f} p50 {np.median(L):.0f} p99 {np.percentile(L, 99):.0f} max {L.max()}; "
      f"warp max steps per tile (max over warps): p50 {np.median(wmax.max(1)):.0f} max {wmax.max()}")
gm = np.array(group_stats)
for k, G in enumerate((32, 64, 128)):
    print(f"warp walk steps with the SIMT max taken per {G}-record group: {gm[:, k].sum()} (SIMT {wsum.sum() / (32 * gm[:, k].sum()):.3f})")
qs_ = np.array(quad_stats)
print(f"1x4 quad steps {qs_[:, 0].sum()} (x{qs_[:, 0].sum() * 4 / cand.sum():.3f} slots/cand), warp max-steps {qs_[:, 1].sum()} "
      f"(2 warps/tile, SIMT {qs_[:, 0].sum() / (32 * qs_[:, 1].sum()):.3f})")
print(f"2x2 quad steps {qs_[:, 2].sum()} (x{qs_[:, 2].sum() * 4 / cand.sum():.3f} slots/cand), warp max-steps {qs_[:, 3].sum()} "
      f"(4 warps x 16 quads: SIMT {qs_[:, 2].sum() / (16 * qs_[:, 3].sum()):.3f})")
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"blend_model_{a.kernel}_{a.mode}.npz"), L=L, last=last,
                    cand=cand, psteps=psteps, wmax=wmax, wsum=wsum, ev=ev, bl=bl,
                    tile=np.array([s[0] for s in stats]))
