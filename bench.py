#!/usr/bin/env python
"""Bench: frames/s and Gaussians/s of the B200 rasterizer at 1080p (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2]

A step renders one 1920x1080 frame of the C2 scene (G(1M, seed 2), SH degree 3,
fitted poly-1 kernel with opacity-aware culling) through ps_render with the scene
resident in HBM. Under torchrun (N > 1) every rank renders its own orbit view of
a replicated scene (view sharding, no data-path collective; "scaling": "weak");
timing is CUDA events on the rasterizer's stream, barrier + max over ranks.
`--impl reference` times the reference's own CPU renderer (oracle/_ref, the
unmodified reference library built from source) on the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/s and Gaussians/s at 1080p, poly-1 vs exp, 1/2/4/8 B200 vs CPU ref"

WORKLOADS = {
    # name: (scene kind, seed, n, width, height, views)
    "c1": ("g", 1, 10_000, 256, 256, 1),
    "c2": ("g", 2, 1_000_000, 1920, 1080, 256),
    "c3": ("g", 4, 6_000_000, 3840, 2160, 1),
    "c4": ("g", 5, 3_000_000, 1920, 1080, 256),
    "c5": ("skewed", 3, 1_000_000, 1920, 1080, 1),
}
HEADLINE = ("poly1/opacity", "poly1", "OpacityAware")
COMPARE = [("exp/stp", "exp", "StopThePop"), ("poly1/zero", "poly1", "ZeroCrossing"),
           ("poly2p/opacity", "poly2p", "OpacityAware"), ("poly3/opacity", "poly3", "OpacityAware")]
# FP32 lane-instructions per kernel evaluation / per blended fragment
OPS_PER_EVAL = {"poly1": 6, "poly2p": 8, "poly3": 8, "exp": 7, "poly2": 8}
OPS_PER_BLEND = 6


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled (every 20 ms) during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "20"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.15)  # first sample lands before the timed region starts
        except OSError:
            self._p = None
        return self

    def __exit__(self, *exc):
        if self._p is None:
            return
        time.sleep(0.05)
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=10)
        except subprocess.TimeoutExpired:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def make_cfg(api, kname: str, mode: str, sh_degree: int):
    return api.RasterConfig(kernel=api.fitted_kernel(kname), culling_mode=getattr(api.CullingMode, mode),
                            sh_degree=sh_degree)


# ---------------------------------------------------------------------------- reference arm
def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle  # the reference's own CPU renderer (oracle/_ref)
    from paper_2603_18707_b200 import api

    kind, seed, n, w, h, _ = WORKLOADS[args.workload]
    ref = oracle.Reference()
    splats, deg = api.synthetic_splat3d({"g": 3, "skewed": 4}[kind], seed, n)
    cam = api.orbit_cameras(256, w, h)[0].to_struct()
    cfg = make_cfg(api, HEADLINE[1], HEADLINE[2], deg).to_struct()
    for _ in range(args.warmup):
        ref.render(splats, cam, cfg)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ref.render(splats, cam, cfg)
        times.append(time.perf_counter() - t0)
    ms = 1000.0 * sum(times) / len(times)
    fps = 1000.0 / ms
    cores = ref.resolve_thread_count(0)
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.workload),
        "gaussians_per_s": fps * n,
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} full frames of {args.workload} ({HEADLINE[0]}) via "
                                   "polysplat::render, OpenMP over all host threads"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(name: str) -> dict:
    kind, seed, n, w, h, views = WORKLOADS[name]
    return {"workload": f"{name.upper()}: synthetic G({n}, seed {seed}{', skewed opacity' if kind == 'skewed' else ''}), "
                        f"{w}x{h}, SH degree 3, {HEADLINE[0]} (fitted poly-1, opacity-aware bound)",
            "gaussians": n, "width": w, "height": h, "kernel": HEADLINE[0], "parallelism": "view-sharded",
            "l2": "flushed between timed steps (256 MiB write); scene (280 MB) also exceeds the 126 MB L2"}


# ---------------------------------------------------------------------------- our arm
def run_ours(args) -> None:
    import numpy as np
    import torch

    from paper_2603_18707_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2603_18707_b200.sharding import max_over_ranks, shard_views

    kind, seed, n, w, h, nviews = WORKLOADS[args.workload]
    scene = api.Scene.synthetic(kind, seed, n)
    deg = scene.sh_degree
    cams = api.orbit_cameras(nviews, w, h)
    if args.workload == "c4":
        # C4: the 256-view batch sharded across ranks every step (scene replicated)
        my_views = list(shard_views(nviews, world, rank))
    else:
        # one view per rank per step (weak scaling); rank 0 renders orbit view 0
        my_views = [(rank * max(1, nviews // max(world, 1))) % nviews]
    cam = cams[my_views[0]]
    frames_per_step = len(my_views)
    r = api.Rasterizer(local)
    ds = r.upload(scene)
    lib = api.lib()
    import ctypes as C
    stream = torch.cuda.ExternalStream(lib.ps_ctx_stream(r.handle), device=torch.device("cuda", local))
    out_rgb = torch.empty((h, w, 3), dtype=torch.float32, device="cuda")
    out_t = torch.empty((h, w), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cam_s = cam.to_struct()

    cam_structs = [cams[v].to_struct() for v in my_views]
    # several views per step: one ps_render_views call (K1 fused over batches of
    # views, each view's binning / blend on its own stream) into per-view outputs
    batch = len(cam_structs) > 1
    if batch:
        cam_arr = (type(cam_structs[0]) * len(cam_structs))(*cam_structs)
        out_rgb = torch.empty((len(cam_structs), h, w, 3), dtype=torch.float32, device="cuda")
        out_t = torch.empty((len(cam_structs), h, w), dtype=torch.float32, device="cuda")

    def render_dev(cfg_s):
        if batch:
            st = lib.ps_render_views(r.handle, ds.handle, cam_arr, len(cam_structs), C.byref(cfg_s),
                                     out_rgb.data_ptr(), out_t.data_ptr(), 1, None)
            if st != 0:
                raise RuntimeError(api.last_error(r.handle))
            return
        for cs in cam_structs:
            st = lib.ps_render(r.handle, ds.handle, C.byref(cs), C.byref(cfg_s), out_rgb.data_ptr(),
                               out_t.data_ptr(), 1, None)
            if st != 0:
                raise RuntimeError(api.last_error(r.handle))

    def timed(cfg_s, steps, warmup, sample_clocks=False):
        for _ in range(warmup):
            render_dev(cfg_s)
        # the timed steps run without per-stage events (events between the
        # kernels would serialise the programmatic dependent launches); the
        # stage split comes from separate frames below
        r.set_timing(False)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        launches = 0
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(local) if sample_clocks else None
        if sampler:
            sampler.__enter__()
        for k in range(steps):
            flush.zero_()
            torch.cuda.synchronize()
            evs[k][0].record(stream)
            render_dev(cfg_s)
            evs[k][1].record(stream)
            launches += r.stats()["kernel_launches"]
        torch.cuda.synchronize()
        if sampler:
            sampler.__exit__(None, None, None)
        ms = sum(a.elapsed_time(b) for a, b in evs) / steps
        ms = max_over_ranks(ms, dist, device="cuda")
        # per-stage split (per frame; a batched step reports its views' summed
        # stage times) from a few more flushed steps with stage events
        r.set_timing(True)
        stage_sum, reps = {}, max(3, min(steps, 20))
        for _ in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            render_dev(cfg_s)
            for key, v in r.stats()["stage_ms"].items():
                stage_sum[key] = stage_sum.get(key, 0.0) + v
        torch.cuda.synchronize()
        r.set_timing(False)
        stages = {k: v / reps / frames_per_step for k, v in stage_sum.items()}
        return ms, stages, launches, (sampler.summary() if sampler else None)

    cfg = make_cfg(api, HEADLINE[1], HEADLINE[2], deg)
    cfg_s = cfg.to_struct()
    ms, stages, launches, clocks = timed(cfg_s, args.steps, args.warmup, sample_clocks=True)
    fps = world * frames_per_step * 1000.0 / ms

    # work counters of the timed frame (untimed render with counters)
    fb_unused, ctr = r.render(ds, cam, cfg, counters=True)
    st = r.stats()
    result = {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
              "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
              "vs_baseline": None, "dtype": "f32 blend, f64 preprocess/binning", "data": "synthetic",
              "config": workload_config(args.workload), "gaussians_per_s": fps * n,
              "gpu_launches": launches, "clocks": clocks}
    result["config"]["views_per_rank_per_step"] = frames_per_step
    result["stages_ms"] = stages
    result["work"] = {"visible": st["visible"], "pairs": st["pairs"], "kernel_evaluations": ctr.kernel_evaluations,
                      "fragments_blended": ctr.fragments_blended, "replay_pixels": st["replay_pixels"],
                      "exact_alpha_evals": st["exact_alpha_evals"]}

    if rank == 0:
        rstages = stages
        if batch:
            # the batched step's per-view stage times overlap across the views'
            # streams; the roofline uses single-view renders of the same workload
            r.set_timing(True)
            acc, reps = {}, 5
            for _ in range(reps):
                flush.zero_()
                torch.cuda.synchronize()
                st_ = lib.ps_render(r.handle, ds.handle, C.byref(cam_structs[0]), C.byref(cfg_s),
                                    out_rgb.data_ptr(), out_t.data_ptr(), 1, None)
                if st_ != 0:
                    raise RuntimeError(api.last_error(r.handle))
                for key, v in r.stats()["stage_ms"].items():
                    acc[key] = acc.get(key, 0.0) + v / reps
            r.set_timing(False)
            rstages = acc
            result["stages_ms_single_view"] = acc
        result["roofline"], result["roofline_stages"] = roofline(r, rstages, n, deg, st, ctr, HEADLINE[1],
                                                                 args.workload)
        if batch:
            result["roofline"]["note"] = "stage times of single-view renders (batched views overlap across streams)"

    # poly-vs-exp and the rest of the kernel matrix (fewer steps each)
    if not args.no_compare:
        kern = {HEADLINE[0]: {"frames_per_s": fps / world, "ms": ms / frames_per_step, "pairs": st["pairs"]}}
        for label, kname, mode in COMPARE:
            c2 = make_cfg(api, kname, mode, deg).to_struct()
            m2, _, _, _ = timed(c2, max(3, min(args.steps, 10)), 3)
            kern[label] = {"frames_per_s": frames_per_step * 1000.0 / m2, "ms": m2 / frames_per_step,
                           "pairs": r.stats()["pairs"] // frames_per_step}  # per view
        # image quality of every kernel against exp / StopThePop (the paper's
        # comparison point), on the device: polysplat::compare (metrics.cpp:138-157)
        ref_cfg = make_cfg(api, "exp", "StopThePop", deg)
        for label, kname, mode in [HEADLINE] + COMPARE:
            if label == "exp/stp":
                continue
            rep = r.compare(ds, cam, ref_cfg, make_cfg(api, kname, mode, deg))
            kern[label].update({"psnr_vs_exp_db": rep.psnr_db, "ssim_vs_exp": rep.ssim,
                                "pair_ratio_vs_exp": rep.pair_ratio})
        result["kernels"] = kern
        result["poly1_vs_exp_speedup"] = kern["exp/stp"]["ms"] / kern[HEADLINE[0]]["ms"]

    # end to end through the public API with host buffers: H2D of the scene
    # from pinned memory + render + D2H of the image, every frame. Two host
    # threads, each with its own context (CUDA stream) and scene copy, as the
    # C ABI's threading model allows, so one frame's H2D overlaps the other's
    # render and D2H (the PCIe H2D of the 280 MB scene is the bound).
    if not args.no_e2e:
        import threading
        pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(scene, k))).pin_memory()
               for k in ("means", "scales", "rotations", "opacities", "sh")}
        r2 = api.Rasterizer(local)
        ds2 = r2.upload(scene)
        lanes = [(r, ds), (r2, ds2)]
        streams = [stream, torch.cuda.ExternalStream(lib.ps_ctx_stream(r2.handle), device=torch.device("cuda", local))]
        outs = [(torch.empty((h, w, 3), dtype=torch.float32).pin_memory(),
                 torch.empty((h, w), dtype=torch.float32).pin_memory()) for _ in lanes]
        ke = max(4, min(args.steps, 12))
        errors = []

        def e2e_frame(li):
            rr, dd = lanes[li]
            hr, ht = outs[li]
            stt = lib.ps_scene_update_soa(rr.handle, dd.handle, pin["means"].data_ptr(), pin["scales"].data_ptr(),
                                          pin["rotations"].data_ptr(), pin["opacities"].data_ptr(),
                                          pin["sh"].data_ptr(), 0)
            if stt != 0:
                raise RuntimeError(api.last_error(rr.handle))
            for cs in cam_structs:
                stt = lib.ps_render(rr.handle, dd.handle, C.byref(cs), C.byref(cfg_s), hr.data_ptr(), ht.data_ptr(),
                                    0, None)
                if stt != 0:
                    raise RuntimeError(api.last_error(rr.handle))

        def worker(li, nframes):
            try:
                for _ in range(nframes):
                    e2e_frame(li)
            except Exception as ex:  # surfaced after join
                errors.append(ex)

        for li in range(len(lanes)):  # warm-up, untimed
            e2e_frame(li)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        streams[1].wait_event(e0)
        per_lane = [ke // 2 + (ke % 2 if li == 0 else 0) for li in range(len(lanes))]
        ths = [threading.Thread(target=worker, args=(li, per_lane[li])) for li in range(len(lanes))]
        for t_ in ths:
            t_.start()
        for t_ in ths:
            t_.join()
        if errors:
            raise errors[0]
        ends = []
        for s_ in streams:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(s_)
            ends.append(ev)
        torch.cuda.synchronize()
        ems = max(e0.elapsed_time(ev) for ev in ends) / ke
        if dist:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        ds2.close()
        r2.close()
        h2d = sum(v.numel() * v.element_size() for v in pin.values())
        result["e2e"] = {"value": world * frames_per_step * 1000.0 / ems, "unit": "frames/s", "ms_per_step": ems,
                         "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(frames_per_step * h * w * 16),
                         "frames_timed": ke,
                         "path": "per frame: ps_scene_update_soa (pinned host SoA) + ps_render (host outputs); "
                                 "2 host threads x 2 contexts, device-timed over all frames"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args.workload, (fb_unused, ctr))

    ds.close()
    r.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def roofline(r, stages: dict, n: int, deg: int, st: dict, ctr, kname: str, workload: str = "c2"):
    """Per-stage achieved vs peak; the dominant stage goes to the top-level `roofline`."""
    import ctypes as C

    from paper_2603_18707_b200 import api

    pk = peaks()
    hbm = float(pk.get("hbm_gbs", 6650.0))
    tf = C.c_double(0)
    api._check(api.lib().ps_measure_fp32_peak(r.handle, C.byref(tf)), r.handle)
    fp32_tflops = tf.value
    v, p = st["visible"], st["pairs"]
    E, B = ctr.kernel_evaluations, ctr.fragments_blended
    sh_bytes = 12 * (deg + 1) ** 2
    work = {  # SURVEY §8(d) algorithmic work per stage
        "preprocess": ("hbm", n * (88 + sh_bytes) + v * 64),
        "duplicate": ("hbm", p * 12),
        "tile_sort": ("hbm", p * 12 * 2),
        "blend": ("fp32", OPS_PER_EVAL.get(kname, 8) * E + OPS_PER_BLEND * B),
    }
    out = {}
    for name, (bound, amount) in work.items():
        ms = stages.get(name, 0.0)
        if ms <= 0:
            continue
        if bound == "hbm":
            ach = amount / (ms * 1e-3) / 1e9
            out[name] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                         "algorithmic": amount, "ms": ms}
        else:
            ach = amount / (ms * 1e-3) / 1e12           # tera FP32 lane-instructions / s
            peak = fp32_tflops / 2.0                     # FFMA = 1 lane-instruction = 2 flops
            out[name] = {"bound": "fp32", "achieved": ach, "peak": peak, "unit": "Tinst/s", "frac": ach / peak,
                         "algorithmic": amount, "ms": ms,
                         "peak_source": f"measured FFMA microbenchmark {fp32_tflops:.1f} TFLOP/s"}
    dom = max(out, key=lambda k: out[k]["ms"]) if out else None
    top = dict(out[dom]) if dom else {}
    if dom:
        top["kernel"] = dom
        top["traffic"], top["traffic_source"] = profiled_traffic(dom, kname, workload)
        if top["bound"] == "hbm":
            top["peak_note"] = ("HBM copy bandwidth from MEASURED_PEAKS.json" if not pk.get("_fallback")
                                else "MEASURED_PEAKS.json absent: B200_PROFILING.md fallback 6650 GB/s")
        else:
            top["peak_note"] = "FP32 issue peak measured in-run (no FP32 entry in MEASURED_PEAKS.json)"
    return top, out


# stage -> kernel-name prefix in the ncu captures (blend: the 16x16 kernel of the headline kernel class)
_STAGE_KERNEL = {"blend": "k_blend16<1, 1, 0", "preprocess": "k_preprocess<3, 1, 3>", "duplicate": "k_duplicate_buckets"}


def profiled_traffic(stage: str, kname: str, workload: str = "c2"):
    """DRAM bytes (read + write) per launch of the stage's kernel, from the
    newest committed `ncu --set full` capture of C2 (profiles/*_ncu_full_c2_raw.csv),
    or (None, reason)."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_full_c2_raw.csv")))
    if not files or kname != "poly1" or stage not in _STAGE_KERNEL or workload != "c2":
        return None, "no matching ncu capture (C2 only)"
    rows = list(csv.reader(open(files[-1])))
    hdr, units = rows[0], rows[1]
    try:
        ki, ri, wi = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    except ValueError:
        return None, "capture lacks dram__bytes metrics"
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[2:]:
        if _STAGE_KERNEL[stage] in r[ki]:
            b = float(r[ri].replace(",", "")) * scale.get(units[ri], 1.0) + \
                float(r[wi].replace(",", "")) * scale.get(units[wi], 1.0)
            return b, f"{os.path.basename(files[-1])} ({r[ki].split('(')[0]})"
    return None, "kernel not in capture"


def full_size_parity(ours, ref_out) -> dict:
    """Our timed frame vs the reference's image of the same frame: max-abs per
    channel and transmittance, PSNR of the white-background composite
    (metrics.cpp:13-44), and the six work counters."""
    import numpy as np
    fb, ctr = ours
    rgb, tr, ctr_ref = ref_out
    d_rgb = float(np.max(np.abs(fb.rgb.astype(np.float64) - rgb)))
    d_t = float(np.max(np.abs(fb.transmittance.astype(np.float64) - tr)))
    ca = fb.rgb.astype(np.float64) + fb.transmittance.astype(np.float64)[..., None]
    cb = rgb + tr[..., None]
    mse = float(np.mean((ca - cb) ** 2))
    return {"max_abs_rgb": d_rgb, "max_abs_t": d_t, "tolerance": 1e-5,
            "psnr_db": None if mse == 0.0 else 10.0 * float(np.log10(1.0 / mse)),
            "counters_identical": ctr.as_dict() == ctr_ref}


def cpu_baseline(workload: str, ours=None) -> dict:
    """The reference's own renderer (oracle/_ref) on this host, bounded sample;
    its image of the frame also checks our timed frame at full size."""
    try:
        from oracle import oracle
        from paper_2603_18707_b200 import api
        kind, seed, n, w, h, _ = WORKLOADS[workload]
        ref = oracle.Reference()
        splats, deg = api.synthetic_splat3d({"g": 3, "skewed": 4}[kind], seed, n)
        cam = api.orbit_cameras(256, w, h)[0].to_struct()
        cfg = make_cfg(api, HEADLINE[1], HEADLINE[2], deg).to_struct()
        ref_out = ref.render(splats, cam, cfg)  # warm-up (its image is the parity check)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            ref.render(splats, cam, cfg)
            ts.append(time.perf_counter() - t0)
        ms = 1000.0 * statistics.median(ts)
        # the reference's stage split: count_pairs = prepare_splats +
        # bin_splats (raster.cpp:310-318); the rest of render is the blend
        tc = []
        for _ in range(3):
            t0 = time.perf_counter()
            ref.count_pairs(splats, cam, cfg)
            tc.append(time.perf_counter() - t0)
        mc = 1000.0 * statistics.median(tc)
        parity = full_size_parity(ours, ref_out) if ours is not None else None
        return {"parity": parity, "value": 1000.0 / ms, "unit": "frames/s", "cores": ref.resolve_thread_count(0), "kind": "reference",
                "ms_per_frame": ms, "stage_split_ms": {"prepare_and_bin": mc, "blend": ms - mc},
                "sample": f"median of 3 full {workload.upper()} frames ({HEADLINE[0]}), "
                          "polysplat::render built from the reference sources, all host threads"}
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": "frames/s", "cores": None, "kind": "reference", "sample": f"unavailable: {e}"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=list(WORKLOADS), default="c2")
    ap.add_argument("--no-compare", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
