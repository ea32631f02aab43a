#!/usr/bin/env python
"""Bench: frames/s and Gaussians/s of the B200 rasterizer at 1080p (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2]

A step renders one 1920x1080 frame of the C2 scene (G(1M, seed 2), SH degree 3,
fitted poly-1 kernel with opacity-aware culling) through ps_render with the scene
resident in HBM (counters off, device outputs: the instantiation
tests/test_gpu_timed_path.py checks against the reference). Under torchrun
(N > 1) every rank renders its own orbit view of a replicated scene each step
(view sharding, no data-path collective; "scaling": "weak"); timing is CUDA
events on the rasterizer's stream, barrier + max over ranks. The line also
carries: the timed frame's parity against the reference's image of the same
frame, the stage split and roofline, the reference's ablation cells with device
times (tools/main.cpp:315-323 + the paper's f'2/S row), the C5 culling ablation,
the C4 256-view batch sharded over the ranks (strong scaling), the end-to-end
rate through the C ABI with host buffers (pinned SoA scene upload, and the
literal drop-in ps_render_splats with a host Splat3D array), and the
reference's own CPU renderer timed on this host.

`--impl reference` times the reference's own CPU renderer (oracle/_ref, the
unmodified reference library built from source) on the same workload, rank 0
only; its inputs come from the reference library too (ref_synth_g /
orbit_cameras), so that arm maps no product code.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
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
# the reference CLI's ablation cells (tools/main.cpp:315-323) + the paper's
# f'2/S row; each is timed on the C2 frame
ABLATION = [("exp/stp", "exp", "StopThePop"), ("poly1/stp", "poly1", "StopThePop"),
            ("poly1/zero", "poly1", "ZeroCrossing"), ("poly1/opacity", "poly1", "OpacityAware"),
            ("poly2p/stp", "poly2p", "StopThePop"), ("poly2p/opacity", "poly2p", "OpacityAware"),
            ("poly3/stp", "poly3", "StopThePop"), ("poly3/opacity", "poly3", "OpacityAware")]
# FP32 lane-instructions per kernel evaluation / per blended fragment
OPS_PER_EVAL = {"poly1": 6, "poly2p": 8, "poly3": 8, "exp": 7, "poly2": 8}
OPS_PER_BLEND = 6
SPLAT3D_BYTES = 59 * 8


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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


def workload_config(name: str) -> dict:
    """The `config` of both arms' lines (identical dicts)."""
    kind, seed, n, w, h, views = WORKLOADS[name]
    return {"workload": f"{name.upper()}: synthetic G({n}, seed {seed}{', skewed opacity' if kind == 'skewed' else ''}), "
                        f"{w}x{h}, SH degree 3, {HEADLINE[0]} (fitted poly-1, opacity-aware bound)",
            "gaussians": n, "width": w, "height": h, "kernel": HEADLINE[0], "parallelism": "view-sharded",
            "views_per_rank_per_step": 1,
            "l2": "flushed between timed steps (256 MiB write); scene (280 MB) also exceeds the 126 MB L2"}


def _scene_key(kind: str) -> int:
    return {"g": 3, "skewed": 4}[kind]


# ---------------------------------------------------------------------------- reference arm
def run_reference(args) -> None:
    """The reference's own CPU renderer (oracle/_ref), rank 0 only. Inputs from
    the reference library itself (ref_synth_g, the reference's orbit_cameras):
    nothing of the product is loaded in this process."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle
    from paper_2603_18707_b200 import abi

    kind, seed, n, w, h, _ = WORKLOADS[args.workload]
    ref = oracle.Reference()
    splats, deg = ref.synth_g(n, seed, kind == "skewed")
    cam = ref.orbit_cameras(256, w, h)[0]
    cfg = abi.default_config()
    cfg.kernel = ref.make_polynomial_kernel(abi.PS_KERNEL_POLY_RELU, (0.77007333317642512, -0.17527402122331368))
    cfg.culling_mode = abi.PS_CULL_OPACITY_AWARE
    cfg.sh_degree = deg
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
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "cpu_model": cpu_model(),
                         "kind": "reference",
                         "sample": f"{args.steps} full frames of {args.workload} ({HEADLINE[0]}) via "
                                   "polysplat::render, OpenMP over all host threads"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm
class Ours:
    """One rank's rasterizer, scene and timing helpers."""

    def __init__(self, args):
        import torch

        from paper_2603_18707_b200 import api
        self.torch, self.api = torch, api
        self.args = args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # PS_BENCH_DEVICE / PS_BENCH_BACKEND=gloo: dry runs of the N > 1 path with
        # every rank on one GPU (tools/runs/r02_bench_n2_dryrun.sh); the driver's
        # runs use one GPU per rank and NCCL
        if os.environ.get("PS_BENCH_DEVICE"):
            self.local = int(os.environ["PS_BENCH_DEVICE"])
        self.backend = os.environ.get("PS_BENCH_BACKEND", "nccl")
        torch.cuda.set_device(self.local)
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
            self.dist = dist
        self.lib = api.lib()
        self.r = api.Rasterizer(self.local)
        self.stream = torch.cuda.ExternalStream(self.lib.ps_ctx_stream(self.r.handle),
                                                device=torch.device("cuda", self.local))
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max_ms(self, ms: float) -> float:
        from paper_2603_18707_b200.sharding import max_over_ranks
        return max_over_ranks(ms, self.dist, device="cuda" if self.backend == "nccl" else "cpu")

    def cfg(self, kname: str, mode: str, deg: int):
        api = self.api
        return api.RasterConfig(kernel=api.fitted_kernel(kname), culling_mode=getattr(api.CullingMode, mode),
                                sh_degree=deg)

    def render_fn(self, ds, cam_structs, cfg_s, out_rgb, out_t):
        """One step's call: ps_render per view (one view) or ps_render_views
        (a batch), counters NULL, device outputs."""
        import ctypes as C
        lib, r, api = self.lib, self.r, self.api
        if len(cam_structs) > 1:
            arr = (type(cam_structs[0]) * len(cam_structs))(*cam_structs)

            def go():
                st = lib.ps_render_views(r.handle, ds.handle, arr, len(cam_structs), C.byref(cfg_s),
                                         out_rgb.data_ptr(), out_t.data_ptr(), 1, None)
                if st != 0:
                    raise RuntimeError(api.last_error(r.handle))
            return go
        cs = cam_structs[0]

        def go1():
            st = lib.ps_render(r.handle, ds.handle, C.byref(cs), C.byref(cfg_s), out_rgb.data_ptr(),
                               out_t.data_ptr(), 1, None)
            if st != 0:
                raise RuntimeError(api.last_error(r.handle))
        return go1

    def timed(self, fn, steps: int, warmup: int, sample_clocks: bool = False):
        """W untimed steps, then K steps each bracketed by CUDA events on the
        rasterizer's stream with an L2 flush before it; barrier + sync on both
        sides; mean ms per step, max over ranks; kernel launches counted."""
        torch = self.torch
        for _ in range(warmup):
            fn()
        self.r.set_timing(False)  # no per-stage events inside the timed steps
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        launches = 0
        self.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(self.local) if sample_clocks else None
        if sampler:
            sampler.__enter__()
        for k in range(steps):
            self.flush.zero_()
            torch.cuda.synchronize()
            evs[k][0].record(self.stream)
            fn()
            evs[k][1].record(self.stream)
            launches += self.r.stats()["kernel_launches"]
        torch.cuda.synchronize()
        self.barrier()
        if sampler:
            sampler.__exit__(None, None, None)
        ms = sum(a.elapsed_time(b) for a, b in evs) / steps
        return self.max_ms(ms), launches, (sampler.summary() if sampler else None)

    def stage_split(self, fn, reps: int, views: int = 1) -> dict:
        """Per-frame stage times (ms) from separate flushed frames with stage events."""
        torch = self.torch
        self.r.set_timing(True)
        acc = {}
        for _ in range(reps):
            self.flush.zero_()
            torch.cuda.synchronize()
            fn()
            for key, v in self.r.stats()["stage_ms"].items():
                acc[key] = acc.get(key, 0.0) + v
        torch.cuda.synchronize()
        self.r.set_timing(False)
        return {k: v / reps / views for k, v in acc.items()}


def run_ours(args) -> None:
    import ctypes as C

    import numpy as np

    o = Ours(args)
    torch, api, lib, r = o.torch, o.api, o.lib, o.r
    world, rank = o.world, o.rank
    kind, seed, n, w, h, nviews = WORKLOADS[args.workload]
    splats = None
    scene = api.Scene.synthetic(kind, seed, n)
    deg = scene.sh_degree
    cams = api.orbit_cameras(nviews, w, h)
    # one view per rank per step (weak scaling); rank 0 renders orbit view 0
    my_view = (rank * max(1, nviews // max(world, 1))) % nviews
    cam = cams[my_view]
    ds = r.upload(scene)
    out_rgb = torch.empty((h, w, 3), dtype=torch.float32, device="cuda")
    out_t = torch.empty((h, w), dtype=torch.float32, device="cuda")
    cfg = o.cfg(HEADLINE[1], HEADLINE[2], deg)
    cfg_s = cfg.to_struct()
    step = o.render_fn(ds, [cam.to_struct()], cfg_s, out_rgb, out_t)

    ms, launches, clocks = o.timed(step, args.steps, args.warmup, sample_clocks=True)
    fps = world * 1000.0 / ms
    # the LAST timed step's image (still in out_rgb / out_t): parity below
    timed_rgb, timed_t = out_rgb.cpu().numpy(), out_t.cpu().numpy()
    stages = o.stage_split(step, max(3, min(args.steps, 20)))
    # work counters of the same frame (the counting instantiation, untimed)
    _, ctr = r.render(ds, cam, cfg, counters=True)
    st = r.stats()
    result = {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
              "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
              "vs_baseline": None, "dtype": "f32 blend, f64 preprocess/binning", "data": "synthetic",
              "config": workload_config(args.workload), "gaussians_per_s": fps * n,
              "gpu_launches": launches, "gpu_launches_per_step": launches / max(args.steps, 1), "clocks": clocks,
              "views_per_rank_per_step": 1, "gpus_active": world}
    result["stages_ms"] = stages
    result["work"] = {"visible": st["visible"], "pairs": st["pairs"], "kernel_evaluations": ctr.kernel_evaluations,
                      "fragments_blended": ctr.fragments_blended, "replay_pixels": st["replay_pixels"],
                      "exact_alpha_evals": st["exact_alpha_evals"]}
    if rank == 0:
        result["roofline"], result["roofline_stages"] = roofline(r, stages, n, deg, st, ctr, HEADLINE[1],
                                                                 args.workload)

    # the reference's ablation cells with device times (f4), and image quality
    # of every cell against exp / StopThePop (polysplat::compare, metrics.cpp:138-157)
    if not args.no_compare:
        ref_cfg = o.cfg("exp", "StopThePop", deg)
        abl = {}
        for label, kname, mode in ABLATION:
            c2 = o.cfg(kname, mode, deg)
            fn = o.render_fn(ds, [cam.to_struct()], c2.to_struct(), out_rgb, out_t)
            m2, _, _ = o.timed(fn, max(3, min(args.steps, 10)), 3)
            sp = o.stage_split(fn, 3)
            _, c_ = r.render(ds, cam, c2, counters=True)
            cell = {"frames_per_s": 1000.0 / m2, "ms": m2, "blend_ms": sp.get("blend", 0.0),
                    "preprocess_ms": sp.get("preprocess", 0.0), "pairs": c_.tile_pairs_after_tight_test,
                    "kernel_evaluations": c_.kernel_evaluations, "fragments_blended": c_.fragments_blended}
            if label != "exp/stp":
                rep = r.compare(ds, cam, ref_cfg, c2)
                cell.update({"psnr_vs_exp_db": rep.psnr_db, "ssim_vs_exp": rep.ssim,
                             "pair_ratio_vs_exp": rep.pair_ratio})
            abl[label] = cell
        result["ablation"] = abl
        result["poly1_vs_exp_speedup"] = abl["exp/stp"]["ms"] / abl[HEADLINE[0]]["ms"]

    # C5 culling ablation: universal (zero-crossing) vs opacity-aware bound on
    # the skewed-opacity scene: key count and blend time (BASELINE.json config 5)
    if not args.no_c5 and args.workload == "c2":
        k5, s5, n5, w5, h5, _ = WORKLOADS["c5"]
        sc5 = api.Scene.synthetic(k5, s5, n5)
        ds5 = r.upload(sc5)
        cam5 = api.orbit_cameras(256, w5, h5)[0]
        c5 = {}
        for label, kname, mode in [("poly1/zero", "poly1", "ZeroCrossing"), ("poly1/opacity", "poly1", "OpacityAware"),
                                   ("exp/stp", "exp", "StopThePop")]:
            cc = o.cfg(kname, mode, sc5.sh_degree)
            fn = o.render_fn(ds5, [cam5.to_struct()], cc.to_struct(), out_rgb, out_t)
            m5, _, _ = o.timed(fn, max(3, min(args.steps, 10)), 3)
            sp = o.stage_split(fn, 3)
            _, c_ = r.render(ds5, cam5, cc, counters=True)
            c5[label] = {"ms": m5, "frames_per_s": 1000.0 / m5, "blend_ms": sp.get("blend", 0.0),
                         "keys": c_.tile_pairs_after_tight_test, "visible": r.stats()["visible"],
                         "fragments_blended": c_.fragments_blended, "kernel_evaluations": c_.kernel_evaluations}
        c5["key_reduction"] = 1.0 - c5["poly1/opacity"]["keys"] / c5["poly1/zero"]["keys"]
        c5["blend_speedup"] = c5["poly1/zero"]["blend_ms"] / max(c5["poly1/opacity"]["blend_ms"], 1e-9)
        result["c5_culling_ablation"] = c5
        ds5.close()
        del sc5

    # C4: the 256-view batch of a 3M scene sharded over the ranks (strong
    # scaling; BASELINE.json config 4): every rank renders its contiguous shard
    # through ps_render_views each step
    if not args.no_c4 and args.workload == "c2":
        from paper_2603_18707_b200.sharding import shard_views
        k4, s4, n4, w4, h4, v4 = WORKLOADS["c4"]
        sc4 = api.Scene.synthetic(k4, s4, n4)
        ds4 = r.upload(sc4)
        cams4 = api.orbit_cameras(v4, w4, h4)
        mine = list(shard_views(v4, world, rank))
        o4_rgb = torch.empty((len(mine), h4, w4, 3), dtype=torch.float32, device="cuda")
        o4_t = torch.empty((len(mine), h4, w4), dtype=torch.float32, device="cuda")
        fn = o.render_fn(ds4, [cams4[v].to_struct() for v in mine], o.cfg("poly1", "OpacityAware", sc4.sh_degree).to_struct(),
                         o4_rgb, o4_t)
        m4, l4, _ = o.timed(fn, max(2, min(args.steps, 3)), 1)
        result["c4_sharded"] = {"views_per_s": v4 * 1000.0 / m4, "ms_per_batch": m4, "views": v4,
                                "views_per_rank": len(mine), "gpus_active": world, "scaling": "strong",
                                "gaussians_per_s": v4 * n4 * 1000.0 / m4, "gpu_launches_per_batch": l4 / max(2, min(args.steps, 3)),
                                "kernel": "poly1/opacity", "path": "ps_render_views per rank, scene replicated, no collective"}
        ds4.close()
        del sc4, o4_rgb, o4_t

    # end to end through the public API with host buffers
    if not args.no_e2e:
        result["e2e"] = e2e_soa(o, scene, ds, [cam.to_struct()], cfg_s, w, h, args)
        splats = api.synthetic_splat3d(_scene_key(kind), seed, n)[0]
        result["e2e_dropin"] = e2e_dropin(o, splats, cam, cfg_s, args)

    if rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(args.workload, (timed_rgb, timed_t, ctr), world)

    ds.close()
    r.close()
    if o.dist:
        o.dist.barrier()
        o.dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def e2e_soa(o, scene, ds, cam_structs, cfg_s, w, h, args) -> dict:
    """Per frame: ps_scene_update_soa from pinned host SoA + ps_render into pinned
    host outputs. Two host threads, each with its own context (CUDA stream) and
    scene copy, as the C ABI's threading model allows, so one frame's H2D
    overlaps the other's render and D2H (the PCIe H2D of the 280 MB scene is the
    bound). Device-timed over all frames."""
    import ctypes as C
    import threading

    import numpy as np
    torch, api, lib, r = o.torch, o.api, o.lib, o.r
    pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(scene, k))).pin_memory()
           for k in ("means", "scales", "rotations", "opacities", "sh")}
    r2 = api.Rasterizer(o.local)
    ds2 = r2.upload(scene)
    lanes = [(r, ds), (r2, ds2)]
    streams = [o.stream, torch.cuda.ExternalStream(lib.ps_ctx_stream(r2.handle), device=torch.device("cuda", o.local))]
    outs = [(torch.empty((h, w, 3), dtype=torch.float32).pin_memory(),
             torch.empty((h, w), dtype=torch.float32).pin_memory()) for _ in lanes]
    ke = max(4, min(args.steps, 12))
    errors = []

    def frame(li):
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
                frame(li)
        except Exception as ex:  # surfaced after join
            errors.append(ex)

    for li in range(len(lanes)):  # warm-up, untimed
        frame(li)
    o.barrier()
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
    ems = o.max_ms(max(e0.elapsed_time(ev) for ev in ends) / ke)
    ds2.close()
    r2.close()
    h2d = sum(v.numel() * v.element_size() for v in pin.values())
    return {"value": o.world * 1000.0 / ems, "unit": "frames/s", "ms_per_step": ems,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(h * w * 16), "frames_timed": ke,
            "path": "per frame: ps_scene_update_soa (pinned host SoA) + ps_render (host outputs); "
                    "2 host threads x 2 contexts, device-timed over all frames"}


def e2e_dropin(o, splats, cam, cfg_s, args) -> dict:
    """The literal drop-in: ps_render_splats (polysplat::b200::render(span<Splat3D>))
    with the reference's host Splat3D array (pageable, 472 B per splat) in and
    an fp64 host framebuffer out, every frame; synchronous call, host wall time."""
    import ctypes as C

    import numpy as np
    api, lib, r = o.api, o.lib, o.r
    a = np.ascontiguousarray(splats, dtype=np.float64)
    cs = cam.to_struct()
    rgb = np.zeros((cam.height, cam.width, 3))
    tr = np.zeros((cam.height, cam.width))
    dp = C.POINTER(C.c_double)

    def call():
        st = lib.ps_render_splats(r.handle, a.ctypes.data_as(dp), len(a), C.byref(cs), C.byref(cfg_s),
                                  rgb.ctypes.data_as(dp), tr.ctypes.data_as(dp), None)
        if st != 0:
            raise RuntimeError(api.last_error(r.handle))

    for _ in range(2):
        call()
    ke = max(3, min(args.steps, 8))
    o.barrier()
    times = []
    for _ in range(ke):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    ms = o.max_ms(1000.0 * statistics.median(times))
    pix = cam.width * cam.height
    h2d = len(a) * 280  # the compact upload record (fp64 geometry + fp32 SH) the host workers write
    d2h = pix * 16 + o.r.stats()["replay_pixels"] * 36
    io_ref = a.nbytes + pix * 32  # the reference interface's bytes: Splat3D array in, fp64 framebuffer out
    return {"value": o.world * 1000.0 / ms, "unit": "frames/s", "ms_per_step": ms, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "frames_timed": ke,
            "interface_bytes_per_step": int(io_ref),
            "pcie_ms_of_interface_bytes_at_53GBps": io_ref / 53e9 * 1e3,
            "vs_pcie_time_of_interface_bytes": ms / (io_ref / 53e9 * 1e3),
            "path": "ps_render_splats: pageable host Splat3D array (472 B/splat) -> host threads narrow it to "
                    "280-B records in a pinned chunk ring -> DMA -> device split + Morton upload -> render -> "
                    "fp32 image + exact replay values -> fp64 host framebuffer; median host wall time of "
                    "synchronous calls"}


def roofline(r, stages: dict, n: int, deg: int, st: dict, ctr, kname: str, workload: str = "c2"):
    """Per-stage achieved vs peak; the dominant stage goes to the top-level `roofline`.
    The blend's time includes its per-tile bucket sort (prologue) and the fused
    exact replay; the tile sort has no separate stage of its own."""
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
    if "blend" in out:
        out["blend"]["includes"] = "per-tile (depth, index) bucket sort in the prologue + fused fp64 replay"
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
_STAGE_KERNEL = {"blend": "k_blend16<1, 1, 0, 0", "preprocess": "k_preprocess<3, 1, 3>", "duplicate": "k_duplicate_buckets"}


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
    """The last timed step's image vs the reference's image of the same frame:
    max-abs per channel and transmittance, PSNR of the white-background
    composite (metrics.cpp:13-44), and the six work counters (of the counting
    render of the same frame)."""
    import numpy as np
    rgb_o, t_o, ctr = ours
    rgb, tr, ctr_ref = ref_out
    d_rgb = float(np.max(np.abs(rgb_o.astype(np.float64) - rgb)))
    d_t = float(np.max(np.abs(t_o.astype(np.float64) - tr)))
    ca = rgb_o.astype(np.float64) + t_o.astype(np.float64)[..., None]
    cb = rgb + tr[..., None]
    mse = float(np.mean((ca - cb) ** 2))
    return {"frame": "last timed step (counter-free blend, device outputs)", "max_abs_rgb": d_rgb, "max_abs_t": d_t,
            "tolerance": 1e-5, "within_tolerance": d_rgb <= 1e-5 and d_t <= 1e-5,
            "psnr_db": None if mse == 0.0 else 10.0 * float(np.log10(1.0 / mse)),
            "counters_identical": ctr.as_dict() == ctr_ref}


def cpu_baseline(workload: str, ours=None, world: int = 1) -> dict:
    """The reference's own renderer (oracle/_ref) on this host, bounded sample;
    its image of the frame also checks our timed frame at full size."""
    try:
        from oracle import oracle
        from paper_2603_18707_b200 import api
        kind, seed, n, w, h, _ = WORKLOADS[workload]
        ref = oracle.Reference()
        splats, deg = ref.synth_g(n, seed, kind == "skewed")
        cam = ref.orbit_cameras(256, w, h)[0]
        cfg = api.RasterConfig(kernel=api.fitted_kernel(HEADLINE[1]),
                               culling_mode=getattr(api.CullingMode, HEADLINE[2]), sh_degree=deg).to_struct()
        ref_out = ref.render(splats, cam, cfg)  # warm-up (its image is the parity check)
        parity = full_size_parity(ours, ref_out) if ours is not None else None
        if world > 1:
            return {"parity": parity, "value": None, "unit": "frames/s", "kind": "reference",
                    "sample": "not timed at N > 1 (rank 0 parity only)"}
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
        return {"parity": parity, "value": 1000.0 / ms, "unit": "frames/s", "cores": ref.resolve_thread_count(0),
                "cpu_model": cpu_model(), "kind": "reference",
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
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
