"""Error-budget model of the blend's exact-replay flags (design-study tool).

Ports the per-splat fp32 error bounds of K1's blend record
(exact_kernels.cu blend_record: Gq, Ga) to numpy, then walks every pixel of
a BASELINE frame with the reference's own prepared splats / tile lists
(oracle/_ref) and predicts which pixels k_blend16 flags:
  * amb   - an accepted fragment with q inside [q* - Gq, q* + Gq];
  * band  - the transmittance interval [Lo, Up] straddling the floor at some step.
Prints the counts and which terms of Ga dominate, so alternative bounds can be
evaluated offline (--scale-gq / --scale-ga multiply the bounds).

    python tools/flag_model.py [--kernel exp --mode StopThePop] [--tiles 4]
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
ap.add_argument("--kernel", default="poly1")
ap.add_argument("--mode", default="OpacityAware")
ap.add_argument("--tiles", type=int, default=1, help="model every k-th tile")
ap.add_argument("--scale-gq", type=float, default=1.0)
ap.add_argument("--scale-ga", type=float, default=1.0)
ap.add_argument("--old", action="store_true", help="round-1 bound (tile-local coordinates, 1e-7 qb)")
ap.add_argument("--centre", action="store_true", help="tile-local arithmetic with the origin at the tile centre")
ap.add_argument("--slack", type=float, default=3.2, help="g' = 1.001 (g + slack u) + 4 u64")
a = ap.parse_args()

e32, e64 = 2.0 ** -24, 2.0 ** -53
ref = oracle.Reference()
splats, deg = ref.synth_g(a.n, a.seed)
cam = ref.orbit_cameras(256, 1920, 1080)[0]
cfg = api.RasterConfig(kernel=api.fitted_kernel(a.kernel), culling_mode=getattr(api.CullingMode, a.mode),
                       sh_degree=deg).to_struct()
prep = ref.prepare(splats, cam, cfg)
off, idx, ctr = ref.tile_lists(splats, cam, cfg)
row = np.full(a.n, -1, np.int64)
row[prep.index] = np.arange(len(prep.index))
k = cfg.kernel
coef = np.array([k.coeffs[j] for j in range(k.order + 1)])
eps, floor = cfg.epsilon, cfg.transmittance_floor
expk = k.kind == 0

# ---- per-splat bounds (blend_record)
ca, cb, cc = prep.conic[:, 0], prep.conic[:, 1], prep.conic[:, 2]
o = prep.opacity_eff
beta = cb / ca
gamma = cc - cb * cb / ca
if expk:
    qs = 2.0 * np.log(o / eps)
else:
    # linear / generic: solve c0 - eps/o + c1 q + ... = 0 numerically (first positive root)
    qs = np.empty_like(o)
    for i in range(len(o)):
        c = coef.copy()
        c[0] -= eps / o[i]
        rts = np.roots(c[::-1])
        rts = rts[(np.abs(rts.imag) < 1e-12) & (rts.real > 0)].real
        qs[i] = rts.min() if len(rts) else 25.0
qb = 1.25 * qs + 1.0 if a.old else 1.01 * qs + 0.01
U, D = np.sqrt(qb / ca), np.sqrt(qb / gamma)
ab_ = np.abs(beta)
X = U + ab_ * D
ts = 16.0
gam_rel = e32 + 4.0 * e64 * (cc + cb * cb / ca) / gamma
if a.old or a.centre:
    tsx = ts / 2 if a.centre else ts
    dmx, dmy = e32 * (X + tsx), e32 * (D + tsx)
    ddx, ddy = dmx + e32 * X, dmy + e32 * D
    du = 2.0 * dmx + ddx + ab_ * ddy + 2.0 * e32 * ab_ * D + e32 * (U + X)
else:
    Mx, My = 0.5 + e32 * (X + ts), 0.5 + e32 * (D + ts)
    dmx, dmy = e32 * Mx, e32 * My
    ddy = dmy + e32 * D
    du = ab_ * ddy + e32 * ab_ * D + dmx + e32 * (ab_ * D + Mx) + e32 * U
dr = qb * (2.0 * e32 + gam_rel) + 2.0 * gamma * D * ddy
dau = qb * 3.0 * e32 + 2.0 * ca * U * du
dq = e32 * qb + dau + dr
refe = 8.0 * e64 * (ca * X * X + 2.0 * np.abs(cb) * X * D + cc * D * D) + 4.0 * e64 * (ca * X + np.abs(cb) * D) * (X + D)
if a.old or expk:
    droot = (1e-7 if a.old else 1e-9) * qb
else:
    pd = sum((j + 1) * coef[j + 1] * qs ** j for j in range(k.order))
    mag = sum(np.abs(coef[j]) * qs ** j for j in range(k.order + 1))
    droot = 1e-9 * qb + 8.0 * e64 * (mag + eps / o) / np.maximum(np.abs(pd), 1e-300)
Gq = (1.25 * (dq + refe) + droot + 1e-12) * a.scale_gq
Gq_terms = {"dau(u)": 1.25 * dau, "dr(row)": 1.25 * dr, "e32 qb": 1.25 * e32 * qb, "droot": droot, "ref": 1.25 * refe}
amax = np.minimum(o if expk else o * coef[0], 0.999)
if expk:
    kp, kmag = 0.5, 0.0
    extra = amax * (2.4e-7 + (0.73 * qb + np.abs(np.log2(o)) + 1.0) * e32 * 0.7)
else:
    d = [coef[1] if k.order >= 1 else 0.0, 2 * coef[2] if k.order >= 2 else 0.0, 3 * coef[3] if k.order >= 3 else 0.0]
    dp = lambda q: np.abs(d[0] + d[1] * q + d[2] * q * q)  # noqa: E731
    kp = np.maximum(dp(0.0), dp(qb))
    kmag = sum(np.abs(coef[j]) * qb ** j for j in range(k.order + 1)) * ((2.0 * k.order + 2.0) if a.old else (k.order + 2.2))
    extra = 0.0
Ga_terms = {"o k' Gq": 1.02 * o * kp * Gq, "eval": 1.02 * e32 * o * kmag, "exp": 1.02 * extra + 0 * o,
            "2u amax": 2.0 * e32 * amax}
Ga = (1.02 * (o * kp * Gq + e32 * o * kmag + extra) + 2.0 * e32 * amax + 1e-15) * a.scale_ga
gp = 1.001 * (Ga + a.slack * e32) + 4.5e-16
print("median Gq terms:", {t: f"{np.median(v):.2e}" for t, v in Gq_terms.items()}, f"Gq {np.median(Gq):.2e}")
print("median Ga terms:", {t: f"{np.median(v):.2e}" for t, v in Ga_terms.items()}, f"Ga {np.median(Ga):.2e}",
      f"g' {np.median(gp):.2e}")

tx_n, ty_n = 120, 68
ly, lx = np.mgrid[0:16, 0:16]
n_amb = n_band = n_px = 0
for t in range(0, tx_n * ty_n, a.tiles):
    lst = idx[off[t]:off[t + 1]]
    L = len(lst)
    if L == 0:
        continue
    r = row[lst]
    tx, ty = t % tx_n, t // tx_n
    gx = (tx * 16 + lx).ravel()
    gy = (ty * 16 + ly).ravel()
    inside = (gx < 1920) & (gy < 1080)
    m = prep.mean2d[r]
    dx = (gx[None, :] + 0.5) - m[:, 0:1]
    dy = (gy[None, :] + 0.5) - m[:, 1:2]
    q = ca[r, None] * dx * dx + 2.0 * cb[r, None] * dx * dy + cc[r, None] * dy * dy
    kv = np.exp(-0.5 * q) if expk else np.maximum(np.polyval(coef[::-1], q), 0.0)
    al = np.minimum(0.999, o[r, None] * kv)
    acc = al >= eps
    amb = acc & (np.abs(q - qs[r, None]) <= Gq[r, None])
    om = np.where(acc, 1.0 - al, 1.0)
    Tb = np.cumprod(np.vstack([np.ones((1, 256)), om[:-1]]), axis=0)
    Tn = Tb * om
    stop = acc & (Tn < floor)
    term = np.where(stop.any(0), stop.argmax(0), L)
    # interval half-width after each step: H' = H (1 - a) + g' T_before  (accepted steps)
    g_step = np.where(acc, gp[r, None], 0.0) * Tb
    H = np.zeros(256)
    band = np.zeros(256, bool)
    ambp = np.zeros(256, bool)
    for j in range(L):
        live = j <= term
        H = H * om[j] + g_step[j]
        hit = live & acc[j] & (np.abs(Tn[j] - floor) <= H)
        band |= hit & ~ambp
        ambp |= live & amb[j] & ~band
        if (j > term).all():
            break
    n_amb += int((ambp & inside).sum())
    n_band += int((band & inside).sum())
    n_px += int(inside.sum())
s = a.tiles
print(f"predicted flags (x{s} tile sampling): amb {n_amb * s}  band {n_band * s}  of {n_px * s} pixels")
