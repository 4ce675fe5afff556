#!/usr/bin/env python3
"""Benchmark of the B200 DRK rasterizer (metric of BASELINE.json: megapixels/s).

Workload (BASELINE.json configs[1], the metric's headline): forward render of
100,000 DRKs, K=8, SH degree 3, 1920x1080, one view per GPU per step
("scaling": "weak": views are independent; primitives replicated; no
data-path collective).  A step goes from raw parameters resident in HBM to the
four framebuffers (colour, depth, normal, alpha) in HBM: activation,
preprocess, tile binning, radix sort, rasterization.  Inputs are seeded
synthetic (paper_2412_11752_b200/scenes.py); L2 is flushed (256 MiB write)
between timed steps and the flush is outside the timed events.

The same line carries:
  e2e          same metric through the C-ABI host-buffer entry (drk_forward_host):
               pinned host params -> H2D -> render -> D2H of all four planes
  fwd_bwd      config 2 (300k DRKs, 1280x720): forward + L1 loss + backward, MP/s
  roofline     dominant kernel (fp32-pass rasterizer): algorithmic FP32 flops
               (SURVEY.md §8(d) counts) / CUDA-event kernel time vs measured FFMA peak
  cpu_baseline the reference CPU renderer (oracle/_ref, unmodified sources) on
               a bounded crop of the same workload, all host threads
`--impl reference` times that reference CPU renderer alone (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# SURVEY.md §8(d) algorithmic FP32 flops (FMA = 2): per pixel, per streamed
# candidate (intersection), per popped candidate (alpha), per composited entry.
F_PIXEL = {0: 34, 3: 82}
F_ISECT = 22
F_ALPHA = 37
F_BLEND = {0: 30, 3: 120}
# Backward, per composited record (grad.cpp:224-301 with backward_alpha
# grad.cpp:16-101, FMA = 2, transcendentals excluded): upstream
# scalar cw 18, rest / dL/dalpha 7, SH 3 + 96 (deg 3) / 3 + 6 (deg 0), normal 6,
# depth 28, backward_alpha 117, (u, v) chain to centre / rotation 57.
F_BWD_RECORD = {0: 240, 3: 330}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-crop", default="960x544", help="crop of the CPU baseline sample (tile aligned)")
    ap.add_argument("--cpu-crop-bwd", default="320x256", help="crop of the CPU fwd+bwd sample (config 2, tile aligned)")
    ap.add_argument("--cpu-crop-c3", default="128x128", help="crop of the CPU config-3 view sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fwd-bwd", action="store_true")
    ap.add_argument("--multiview-views", type=int, default=64,
                    help="config 3 leg: orbit views per step, split across ranks (0 = skip)")
    ap.add_argument("--multiview-inflight", type=int, default=1,
                    help="config 3 leg: rasterizer contexts in flight per GPU (own stream + host thread each)")
    ap.add_argument("--no-config4-train", action="store_true",
                    help="skip the config-4 training step (4M DRK, 8 views of 3840x2160 per GPU; ~1 min)")
    ap.add_argument("--no-adapter", action="store_true", help="skip the drop-in adapter leg (drk::render / "
                    "drk::backward_render through oracle/_ref/adapter_bench)")
    ap.add_argument("--no-train", action="store_true", help="skip the multi-GPU training-step leg")
    return ap.parse_args()


def maybe_spawn(args) -> None:
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run
    with N ranks (one per GPU, rendezvous on 127.0.0.1); the driver's own torchrun
    launch sets WORLD_SIZE and runs the ranks directly."""
    if "WORLD_SIZE" in os.environ or args.gpus <= 1:
        return
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


_JSON_FD = None


def claim_stdout() -> None:
    """Keep stdout for the one JSON line: anything else written to file
    descriptor 1 (NCCL's version banner, library prints) goes to stderr."""
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


def emit(line: dict) -> None:
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.lines, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def reference_cpu_sample(crop: str, steps: int = 1):
    """Reference CPU forward (activate + render, all host threads) on a centred crop of config 1."""
    from oracle import ref
    from paper_2412_11752_b200 import scenes
    w, h = (int(x) for x in crop.split("x"))
    sc = scenes.config_scene(1)
    cam0 = scenes.config_cameras(1)[0]
    x0 = (cam0.width // 2 - w // 2) // 16 * 16
    y0 = (cam0.height // 2 - h // 2) // 16 * 16
    cam = cam0.crop(x0, y0, w, h)
    threads = ref.hardware_threads()
    opt = ref.Options(sh_degree=3, threads=0)
    secs = []
    for _ in range(steps):
        secs.append(ref.render(sc, cam, opt)["seconds"])
    t = float(np.mean(secs))
    return dict(value=w * h / t / 1e6, unit="megapixels/s", cores=threads, kind="reference",
                sample=f"config 1 (100k DRK, SH3) centred {w}x{h} crop of the 1920x1080 view; reference activate+render "
                       f"(oracle/_ref, unmodified sources, -O3) with RenderOptions::threads=0 ({threads} threads); "
                       f"bin_primitives (single-threaded by design) still processes all primitives; "
                       f"{steps} run(s), {t:.2f} s each"), t


def reference_cpu_fwd_bwd(crop: str):
    """Reference CPU training-step span on a centred crop of config 2: activate + render(&replay)
    + L1 loss + backward_render (oracle/_ref ref_fwd_bwd), all host threads."""
    from oracle import ref
    from paper_2412_11752_b200 import scenes
    w, h = (int(x) for x in crop.split("x"))
    sc = scenes.config_scene(2)
    cam0 = scenes.config_cameras(2)[0]
    cam = cam0.crop((cam0.width // 2 - w // 2) // 16 * 16, (cam0.height // 2 - h // 2) // 16 * 16, w, h)
    out = ref.fwd_bwd(sc, cam, scenes.config_target(2, cam), ref.Options(sh_degree=3, threads=0))
    t = out["seconds_fwd"] + out["seconds_bwd"]
    threads = ref.hardware_threads()
    return dict(value=w * h / t / 1e6, unit="megapixels/s", cores=threads, kind="reference",
                seconds_fwd=out["seconds_fwd"], seconds_loss_bwd=out["seconds_bwd"],
                sample=f"config 2 (300k DRK, SH3) centred {w}x{h} crop of the 1280x720 view; reference activate + "
                       f"render(&replay) + L1 loss + backward_render (oracle/_ref, unmodified sources) with "
                       f"threads=0 ({threads} threads); bin_primitives (single-threaded) still processes all "
                       f"primitives; {t:.2f} s")


def reference_cpu_config3(crop: str):
    """Reference CPU forward of one config-3 orbit view (1M DRK) on a centred crop, all host threads."""
    from oracle import ref
    from paper_2412_11752_b200 import scenes
    w, h = (int(x) for x in crop.split("x"))
    sc = scenes.config_scene(3)
    cam0 = scenes.config_cameras(3)[0]
    cam = cam0.crop((cam0.width // 2 - w // 2) // 16 * 16, (cam0.height // 2 - h // 2) // 16 * 16, w, h)
    t = ref.render(sc, cam, ref.Options(sh_degree=3, threads=0))["seconds"]
    threads = ref.hardware_threads()
    return dict(value=w * h / t / 1e6, unit="megapixels/s", cores=threads, kind="reference", seconds=t,
                sample=f"config 3 (1M DRK, SH3) view 0, centred {w}x{h} crop of the 1920x1080 view; reference "
                       f"activate + render with threads=0 ({threads} threads); bin_primitives (single-threaded) "
                       f"still processes all 1M primitives, which dominates a crop this small; {t:.2f} s")


def adapter_leg(warm: int = 1, steps: int = 3):
    """drk::render / drk::loss / drk::backward_render through the drop-in adapter
    (oracle/_ref/adapter_bench, DRK_ADAPTER_PRECISION=fast) on config 2: host
    std::vector<DrkPrimitive> in, host Images / ParamGrads out."""
    import tempfile

    from paper_2412_11752_b200 import scenes
    exe = os.path.join(ROOT, "oracle", "_ref", "adapter_bench")
    if not os.path.exists(exe):
        return {"unavailable": "oracle/_ref/adapter_bench not built"}
    sc = scenes.config_scene(2)
    cam = scenes.config_cameras(2)[0]
    tgt = scenes.config_target(2, cam)
    with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as fh:
        fh.write(np.array([sc.n, sc.k, sc.terms, cam.width, cam.height], np.int32).tobytes())
        fh.write(np.concatenate([[cam.fx, cam.fy, cam.cx, cam.cy], np.asarray(cam.R).ravel(),
                                 np.asarray(cam.t).ravel()]).astype(np.float64).tobytes())
        fh.write(sc.f32().tobytes())
        fh.write(np.ascontiguousarray(tgt, np.float64).tobytes())
        path = fh.name
    try:
        env = dict(os.environ, DRK_ADAPTER_PRECISION="fast")
        rr = subprocess.run([exe, path, str(warm), str(steps)], capture_output=True, text=True, timeout=600, env=env)
        if rr.returncode != 0:
            return {"unavailable": f"adapter_bench rc={rr.returncode}: {rr.stderr[-300:]}"}
        res = json.loads(rr.stdout.strip().splitlines()[-1])
    finally:
        os.unlink(path)
    px = cam.width * cam.height
    return {"render": {"value": px / (res["render_ms"] * 1e-3) / 1e6, "unit": "megapixels/s",
                       "ms_per_step": res["render_ms"]},
            "fwd_bwd": {"value": px / (res["render_loss_backward_ms"] * 1e-3) / 1e6, "unit": "megapixels/s",
                        "ms_per_step": res["render_loss_backward_ms"]},
            "activate_ms_host": res["activate_ms"], "steps": res["steps"],
            "workload": "config 2 (300k DRK, SH3, 1280x720) through the reference C++ API: drk::render, then "
                        "drk::render + drk::loss (L1) + drk::backward_render (deterministic parallel backward), "
                        "host std::vector<DrkPrimitive> in / host Images and ParamGrads out (conversions and copies "
                        "timed; drk::activate on the host, reported apart)"}


def run_reference(args):
    """Reference CPU arm: rank 0 alone times the unmodified reference (oracle/_ref): W untimed
    warm-up samples, then K bounded samples timed (~5 s each on 16 host threads)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    for _ in range(max(0, args.warmup)):
        reference_cpu_sample(args.cpu_crop, 1)
    vals, cpu = [], None
    for _ in range(max(1, args.steps)):
        cpu, _ = reference_cpu_sample(args.cpu_crop, 1)
        vals.append(cpu["value"])
    v = float(np.mean(vals))
    cpu["value"] = v
    w, h = (int(x) for x in args.cpu_crop.split("x"))
    fb = reference_cpu_fwd_bwd(args.cpu_crop_bwd)
    line = {"impl": "reference", "metric": "megapixels/sec rendered (forward; fwd+bwd in fwd_bwd)", "value": v,
            "unit": "megapixels/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * (w * h) / (v * 1e6), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded scenes.py generator)",
            "config": {"workload": f"config1 forward (100k DRK, K=8, SH3, 1920x1080 view), {args.cpu_crop} centred "
                                   "crop per step as the bounded CPU sample", "primitives": 100000, "K": 8,
                       "sh_degree": 3},
            "cpu_baseline": cpu,
            "fwd_bwd": {"value": fb["value"], "unit": "megapixels/s", "ms_per_step": 1e3 * (fb["seconds_fwd"] +
                                                                                           fb["seconds_loss_bwd"]),
                        "workload": fb["sample"]},
            "e2e": {"value": v, "unit": "megapixels/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def main():
    args = parse()
    maybe_spawn(args)
    claim_stdout()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    from paper_2412_11752_b200 import scenes
    from paper_2412_11752_b200.api import FrameGrad, Rasterizer, RenderOptions

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    r = Rasterizer(local)
    r.set_timing(True)
    cfg = 1
    sc = scenes.config_scene(cfg)
    cam = scenes.config_cameras(cfg)[0]
    opt = RenderOptions(sh_degree=3)
    raw = torch.from_numpy(sc.f32()).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    r.set_counters(True)
    for _ in range(args.warmup):
        r.render(raw, cam, opt)
    torch.cuda.synchronize(dev)
    # the warm-up frames ran with the work counters on: they give the roofline's
    # counts (the frame is deterministic); the timed frames run without them
    stats0 = r.stats()
    r.set_counters(False)

    # ---- device-resident timed region ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    raster_ms, launches, stage_acc = [], 0, {}
    barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            r.render(raw, cam, opt)
            evs[i][1].record(stream)
            st = r.stats()
            raster_ms.append(st["stage_ms"]["raster"])
            launches += st["launches"]
            for k, v in st["stage_ms"].items():
                stage_acc[k] = stage_acc.get(k, 0.0) + v
        torch.cuda.synchronize(dev)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tot_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    px = cam.width * cam.height
    value = world * px / (ms_per_step * 1e-3) / 1e6
    st = stats0

    # ---- roofline of the dominant kernel (fp32-pass rasterizer) ----
    flops = (px * F_PIXEL[3] + st["streamed"] * F_ISECT + st["popped"] * F_ALPHA + st["composited"] * F_BLEND[3])
    rast_ms = float(np.mean(raster_ms))
    peak = r.fp32_peak_tflops()
    achieved = flops / (rast_ms * 1e-3) / 1e12
    stage_ms = {k: v / args.steps for k, v in stage_acc.items() if k in ("activate", "preprocess", "rows_emit", "sort",
                                                                         "raster", "raster_fp64")}
    traffic, traffic_src, pipes = None, None, None
    try:  # DRAM bytes of the dominant kernel from the committed ncu --set full capture (profiles/)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tj = json.load(fh)
            traffic = tj.get("k_raster_fast")
            traffic_src = tj.get("source", "profiles/ncu_traffic.json")
            pipes = tj.get("k_raster_fast_pipes")
    except (OSError, ValueError):
        traffic, pipes = None, None
    roofline = {"kernel": "k_raster_fast (fp32 interval pass)", "bound": "fp32", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_source": f"committed ncu --set full capture (not measured in this run): {traffic_src}",
                "peak_source": "FFMA microbenchmark (drk_measure_fp32_peak) in this run; MEASURED_PEAKS.json has no "
                               "FP32 CUDA-core figure",
                "algorithmic_flops_per_launch": flops, "kernel_ms": rast_ms,
                "pipe_utilisation": pipes,
                "counts": {"pixels": px, "streamed": st["streamed"], "popped": st["popped"],
                           "composited": st["composited"]},
                "share_of_step": rast_ms / ms_per_step}
    # ---- HBM stages of the same frame: algorithmic bytes / CUDA-event stage time ----
    hbm_peak, hbm_src = 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hbm_peak, hbm_src = float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        pass
    S1 = sc.raw.shape[0]
    algo_bytes = {
        "activate": sc.n * (4 * S1 + 4 * 79),   # raw f32 in, activated record (79 values) out
        "preprocess": sc.n * (8 * 31 + 160),    # activated fp64 geometry in, 160-B screen record out
        "rows_emit": st["pairs"] * 12,          # one (u64 key, u32 id) pair written per tile entry
        "sort": st["pairs"] * 16,               # u32 key + u32 id written once and read once
    }
    hbm_stages = {}
    for k, b in algo_bytes.items():
        ms = stage_ms.get(k, 0.0)
        gbs = b / (ms * 1e-3) / 1e9 if ms else None
        hbm_stages[k] = {"bytes": int(b), "ms": ms, "GB/s": gbs, "frac": gbs / hbm_peak if gbs else None}
    hbm_roofline = {"bound": "hbm", "peak": hbm_peak, "unit": "GB/s", "peak_source": hbm_src, "stages": hbm_stages,
                    "note": "K1 preprocess and K2 rows+emit are FP64 / latency bound (wedge polygons, fp64 keys), "
                            "so their HBM fractions are low by construction; the sort is the HBM-bound stage"}

    # ---- e2e through the C-ABI host-buffer entry ----
    e2e = None
    host_raw = torch.from_numpy(sc.f32()).pin_memory()
    outs = {"color": torch.empty(cam.height, cam.width, 3, pin_memory=True),
            "depth": torch.empty(cam.height, cam.width, pin_memory=True),
            "normal": torch.empty(cam.height, cam.width, 3, pin_memory=True),
            "alpha": torch.empty(cam.height, cam.width, pin_memory=True)}
    for _ in range(max(1, args.warmup)):
        r.render_host_ptrs(host_raw, outs, cam, opt)
    torch.cuda.synchronize(dev)
    barrier()
    e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r.render_host_ptrs(host_raw, outs, cam, opt)
        b.record(stream)
        b.synchronize()
        e_ms.append(a.elapsed_time(b))
    e_tot = float(np.sum(e_ms))
    if world > 1:
        t = torch.tensor([e_tot], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_tot = float(t.item())
    e2e = {"value": world * px / (e_tot / args.steps * 1e-3) / 1e6, "unit": "megapixels/s",
           "h2d_bytes_per_step": int(host_raw.numel() * 4), "d2h_bytes_per_step": int(px * 8 * 4),
           "path": "drk_forward_host (C-ABI): pinned host raw params -> device (H2D copy) -> render; the raster "
                   "kernels store the 4 framebuffers into the pinned host buffers (zero-copy D2H)"}

    # ---- forward + backward (config 2) ----
    fwd_bwd = None
    if not args.no_fwd_bwd:
        sc2 = scenes.config_scene(2)
        cam2 = scenes.config_cameras(2)[0]
        raw2 = torch.from_numpy(sc2.f32()).to(dev)
        tgt2 = torch.from_numpy(scenes.config_target(2, cam2).astype(np.float32)).to(dev)
        opt2 = RenderOptions(sh_degree=3)
        grad2 = torch.zeros_like(raw2)

        def train_step():
            fb = r.render(raw2, cam2, opt2)
            _, dcol = r.l1_loss(fb.color, tgt2)
            r.backward_render(raw2, FrameGrad(d_color=dcol), grad_out=grad2)

        r.set_counters(True)  # one counted frame (deterministic): the backward roofline's work counts
        train_step()
        st2 = r.stats()
        r.set_counters(False)
        for _ in range(max(1, min(args.warmup, 2))):
            train_step()
        torch.cuda.synchronize(dev)
        nfb = max(2, args.steps // 2)
        fb_ms = []
        bst = {}
        for _ in range(nfb):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            train_step()
            b.record(stream)
            b.synchronize()
            fb_ms.append(a.elapsed_time(b))
            s2 = r.stats()["stage_ms"]
            for k, v in s2.items():
                bst[k] = bst.get(k, 0.0) + v / nfb
        fb_tot = float(np.mean(fb_ms))
        if world > 1:
            t = torch.tensor([fb_tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            fb_tot = float(t.item())
        px2 = cam2.width * cam2.height
        bwd_ms = bst.get("backward_raster", 0.0)
        bflops = (px2 * F_PIXEL[3] + st2["streamed"] * F_ISECT + st2["popped"] * F_ALPHA
                  + st2["composited"] * (F_BLEND[3] + F_BWD_RECORD[3]))
        roofline_bwd = {"kernel": "k_raster_bwd_fast + fp64 pixel backward (stage backward_raster)", "bound": "fp32",
                        "achieved": bflops / (bwd_ms * 1e-3) / 1e12 if bwd_ms else None, "peak": peak,
                        "unit": "TFLOP/s", "frac": (bflops / (bwd_ms * 1e-3) / 1e12) / peak if bwd_ms else None,
                        "algorithmic_flops_per_launch": bflops, "kernel_ms": bwd_ms,
                        "counts": {"pixels": px2, "streamed": st2["streamed"], "popped": st2["popped"],
                                   "composited_records": st2["composited"]},
                        "per_unit": {"pixel": F_PIXEL[3], "streamed": F_ISECT, "popped": F_ALPHA,
                                     "record": F_BLEND[3] + F_BWD_RECORD[3]},
                        "share_of_step": bwd_ms / fb_tot if fb_tot else None}
        fwd_bwd = {"value": world * px2 / (fb_tot * 1e-3) / 1e6, "unit": "megapixels/s", "ms_per_step": fb_tot,
                   "steps": nfb, "workload": "config2: 300k DRK, K=8, SH3, 1280x720, forward + L1 loss + backward "
                                             "(raw-parameter gradients), one view per GPU",
                   "stage_ms": bst, "roofline_bwd": roofline_bwd}

    # ---- config 3: multi-view batch, views sharded across ranks (strong scaling) ----
    multiview = None
    if args.multiview_views > 0:
        from paper_2412_11752_b200.parallel import shard_views
        sc3 = scenes.config_scene(3)
        cams3 = scenes.config_cameras(3)[:args.multiview_views]
        raw3 = torch.from_numpy(sc3.f32()).to(dev)
        from paper_2412_11752_b200.parallel import MultiViewRenderer
        # per-view cost = tile pairs, from one pass over views v = rank (mod world),
        # gathered so that every rank shards the same way (greedy LPT, shard_views)
        cost = torch.zeros(len(cams3), dtype=torch.float64, device=dev)
        for i, v in enumerate(range(rank, len(cams3), world)):
            if i == 0:
                r.render(raw3, cams3[v], opt)
            else:
                r.render_again(cams3[v], opt)
            cost[v] = float(r.stats()["pairs"])
        if world > 1:
            dist.all_reduce(cost)
        mine = shard_views(len(cams3), world, rank, cost.cpu().numpy())
        my_cams = [cams3[v] for v in mine]
        mvr = MultiViewRenderer(local, inflight=args.multiview_inflight)
        for rr in mvr.rasts:
            rr.set_counters(False)
        mvr.render(raw3, my_cams, opt)  # warm-up pass over this rank's views (buffers reach their peak sizes)
        torch.cuda.synchronize(dev)
        nmv = max(1, min(args.steps, 2))
        mv_ms = []
        for _ in range(nmv):
            barrier()
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            mvr.render(raw3, my_cams, opt)  # joins its streams back into `stream` before returning
            b.record(stream)
            b.synchronize()
            mv_ms.append(a.elapsed_time(b))
        mv_tot = float(np.mean(mv_ms))
        if world > 1:
            t = torch.tensor([mv_tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            mv_tot = float(t.item())
        px3 = cams3[0].width * cams3[0].height
        multiview = {"value": len(cams3) * px3 / (mv_tot * 1e-3) / 1e6, "unit": "megapixels/s",
                     "ms_per_step": mv_tot, "steps": nmv, "scaling": "strong", "views_per_step": len(cams3),
                     "views_on_rank0": len(mine), "inflight_contexts": args.multiview_inflight,
                     "sharding": "greedy longest-first by tile-pair count (shard_views), pairs gathered over ranks",
                     "workload": f"config3: 1M DRK, K=8, SH3, {len(cams3)} of the 64 seeded orbit views at 1920x1080 "
                                 "per step, views split across ranks by cost (replicated primitives, no data-path collective); "
                                 "on each GPU the primitives are activated once per step and the views stream through "
                                 "MultiViewRenderer (in-flight contexts: --multiview-inflight); max over ranks"}
        mvr.close()
        del raw3

    # ---- training step: per-rank views, NCCL all-reduce of the raw gradients, Adam (config 4 structure at
    #      config 2 scale: 300k DRK, 1280x720, 2 views per GPU) ----
    train = None

    def train_leg(cfg_id: int, views_per_gpu: int, warm: int, timed: int):
        """Training step: per-rank views, forward + L1 + backward per view (raw gradients
        accumulated), NCCL all-reduce (mean over all views), Adam; max over ranks."""
        from paper_2412_11752_b200.api import OptState, TrainConfig
        from paper_2412_11752_b200.parallel import NcclComm, params_checksum
        sc_t = scenes.config_scene(cfg_id)
        base_cam = scenes.config_cameras(cfg_id)[0]
        orbit = scenes.orbit_cameras(views_per_gpu * world, base_cam.width, base_cam.height, seed=4)
        views = orbit[views_per_gpu * rank:views_per_gpu * (rank + 1)]
        tg = [torch.from_numpy(scenes.config_target(cfg_id, cv, view=views_per_gpu * rank + i).astype(np.float32))
              .to(dev) for i, cv in enumerate(views)]
        p_t = torch.from_numpy(sc_t.f32()).to(dev)
        del sc_t
        g_t = torch.zeros_like(p_t)
        st_t = OptState.zeros_like(p_t)
        tcfg = TrainConfig(steps=35000, lr_drk=1e-3, lr_position=1e-3 / 2.0, lr_rotation=1e-3, lr_opacity=1e-3,
                           lr_sh=1e-3)
        opt_t = RenderOptions(sh_degree=3)
        comm = NcclComm(r, rank, world)

        def step():
            g_t.zero_()
            for cv, tgt in zip(views, tg):
                fb = r.render(p_t, cv, opt_t)
                _, dcol = r.l1_loss(fb.color, tgt)
                r.backward_render(p_t, FrameGrad(d_color=dcol), grad_out=g_t, accumulate=True)
            # native NCCL exchange: reduce-scatter (sum), Adam on this rank's shard
            # with the 1 / total-views scale folded in, all-gather of the parameters
            r.allreduce_adam(comm, p_t, g_t, st_t, tcfg, scene_extent=2.0, grad_scale=1.0 / (views_per_gpu * world))

        for _ in range(warm):
            step()
        torch.cuda.synchronize(dev)
        tr_ms = []
        for _ in range(timed):
            barrier()
            torch.cuda.synchronize(dev)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            b.synchronize()
            tr_ms.append(a.elapsed_time(b))
        tr_tot = float(np.mean(tr_ms))
        csum = params_checksum(p_t)
        in_sync = True
        if world > 1:
            t = torch.tensor([tr_tot], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tr_tot = float(t.item())
            cs = torch.tensor([csum, -csum], device=dev, dtype=torch.float64)
            dist.all_reduce(cs, op=dist.ReduceOp.MAX)
            in_sync = bool(abs(float(cs[0].item()) + float(cs[1].item())) == 0.0)
        px = base_cam.width * base_cam.height
        comm.close()
        return {"value": views_per_gpu * world * px / (tr_tot * 1e-3) / 1e6, "unit": "megapixels/s",
                "ms_per_step": tr_tot, "steps": timed, "warmup": warm, "scaling": "weak", "replicas_in_sync": in_sync,
                "exchange": "drk_allreduce_adam (native NCCL: reduce-scatter, sharded Adam, all-gather)"}

    if not args.no_train:
        train = train_leg(2, 2, 1, 2)
        train["workload"] = ("training step with config 4's structure at config 2 scale: 300k DRK, K=8, SH3, 2 orbit "
                             "views of 1280x720 per GPU, forward + L1 + backward per view, NCCL reduce-scatter of the raw "
                             "gradients, Adam (lr 1e-3, mean over all views) on each rank's shard, all-gather; "
                             "replicas checked by parameter checksum")
    train_c4 = None
    if not args.no_config4_train:
        train_c4 = train_leg(4, 8, 1, 1)
        train_c4["workload"] = ("config 4 training step: 4M DRK, K=8, SH3, 8 orbit views of 3840x2160 per GPU "
                                "(banded binning), forward + L1 + backward per view, NCCL reduce-scatter of the raw "
                                "gradients, Adam (lr 1e-3, mean over all views) on each rank's shard, all-gather; one "
                                "warm-up step (buffer growth)")

    # ---- drop-in adapter (rank 0, N = 1): the reference C++ API served by the GPU ----
    adapter = None
    if rank == 0 and world == 1 and not args.no_adapter:
        adapter = adapter_leg()

    # ---- CPU baseline (rank 0, N = 1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu, _ = reference_cpu_sample(args.cpu_crop, 1)
            cpu["fwd_bwd"] = reference_cpu_fwd_bwd(args.cpu_crop_bwd)
            cpu["config3_view"] = reference_cpu_config3(args.cpu_crop_c3)
        except Exception as e:  # the oracle build is missing: report, do not fail the bench
            cpu = {"value": None, "unit": "megapixels/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {"metric": "megapixels/sec rendered (forward; fwd+bwd in fwd_bwd)", "value": value,
                "unit": "megapixels/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32 (fp32 tile-linearised intersections and alpha with error bounds; fp64 at ties, sort keys "
                         "and transmittance)",
                "data": "synthetic (seeded scenes.py generator; BASELINE.json config 1 distributions)",
                "config": {"workload": "config1 forward: 100k DRK, K=8, SH degree 3, 1920x1080, 1 view per GPU per step",
                           "primitives": 100000, "K": 8, "sh_degree": 3, "width": 1920, "height": 1080,
                           "views_per_gpu": 1, "parallelism": f"views x{world} (replicated primitives)",
                           "l2": "flushed between timed steps (256 MiB write, outside the timed events)"},
                "stage_ms": stage_ms, "pairs": st["pairs"], "fp64_pixels": st["fp64_pixels"],
                "roofline": roofline, "hbm_roofline": hbm_roofline, "adapter": adapter, "e2e": e2e, "fwd_bwd": fwd_bwd, "multiview": multiview, "train": train, "train_config4": train_c4,
                "cpu_baseline": cpu,
                "clocks": clk.summary(), "gpu_launches": int(launches)}
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
