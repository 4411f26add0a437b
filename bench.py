"""Benchmark: streaming FPS & per-block latency of the TPP/RSFM denoiser hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 14b|1.3b] [--impl ours|reference]

One "step" = one streamed block (3 latent frames -> 12 video frames) through
all T=4 denoising steps of the Wan-shaped causal DiT with the RSFM sink and
full rolling KV caches (L=4: N_kv = 1560 + 4*4680 + 4680 = 24960 keys per
layer).  N=1 runs the T steps sequentially on one B200;
N>1 runs TPP stages across GPUs (see tpp_dist.py), one process per GPU.

Synthetic data: random-init weights of the named shape drawn on the device,
N(0,1) noise blocks, synthetic audio/prompt features.  Inputs (weights
19.7 GB, KV caches 4 x 20.4 GB at 14B) are far larger than the 126 MB L2,
so no L2 flush is needed between steps.

`value` = FPS with the noise resident in HBM; `e2e` = the same through the
StreamingPipeline API with the noise copied from pinned host memory and the
denoised latent read back, per step, inside the timed region.
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

FRAMES_PER_BLOCK_VIDEO = 12  # 3 latent frames x 4 (VAE temporal upsampling), BASELINE.md
METRIC = "streaming FPS & per-block latency, 14B-shape 4-step TPP, at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="14b", choices=["14b", "1.3b"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--no-decode", action="store_true", help="skip the decode-stage measurement (clean ncu launch lists)")
    ap.add_argument("--decode-gpu", action="store_true",
                    help="N>1: one dedicated decode rank per pipeline (the paper's 4 DiT + 1 VAE layout)")
    ap.add_argument("--history-sigma", type=float, default=0.0,
                    help="history-noise sigma (config 4: corrupted cache views, device Philox noise)")
    ap.add_argument("--api", default="stream", choices=["stream", "dropin"],
                    help="dropin: the reference-facing B200Denoiser.denoise_block loop (host latents per call, "
                         "the reference engine's run_sequential driving order) instead of the streaming engine")
    ap.add_argument("--long-horizon", type=int, default=0, metavar="BLOCKS",
                    help="config 4: one stream of BLOCKS blocks (834 = 10k video frames) from a cold start: "
                         "whole-run and steady FPS, measured TTFF, per-block latency, drift, ring replay")
    ap.add_argument("--history-mode", default="fixed", choices=["fixed", "scaled"])
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo lets several ranks share one GPU in tests)")
    return ap.parse_args()


def profile_for(name):
    from paper_2512_04677_b200.model import WAN_14B, WAN_1_3B

    return WAN_14B if name == "14b" else WAN_1_3B


def workload_config(args):
    """The workload definition every arm of this bench reports as ``config``
    (ours at any N and the reference arm): identical dicts for one command."""
    prof = profile_for(args.config)
    n_tok = 3 * prof.tokens_per_frame
    return {"workload": workload(args.config), "steps_T": 4, "cache_L": 4, "tokens_per_block": n_tok,
            "n_kv_steady": prof.tokens_per_frame + 4 * n_tok + n_tok, "history_sigma": args.history_sigma,
            "l2": "inputs (weights + KV rings) >> 126 MB L2; no flush needed"}


def workload(name):
    return {"14b": "Wan-14B-shape causal DiT (40 layers, dim 5120, 40 heads, ffn 13824), 4-step, 480p block",
            "1.3b": "Wan-1.3B-shape causal DiT (30 layers, dim 1536, 12 heads, ffn 8960), 4-step, 480p block"}[name]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_baseline(prof, n_tok, n_kv, steps, target_s=10.0):
    """The reference algorithm on the host cores: its pinned-order
    numerics.matmul (99.4% of denoise_block at 14B dims) on a
    bounded K-slice at this token count, extrapolated linearly in FLOPs to a
    whole block (labelled "extrapolated")."""
    from oracle.cpu_bench import pinned_matmul_rate

    r = pinned_matmul_rate(n_tok, prof.model_dim, k_slice=32, target_s=target_s)
    flops_block = steps * prof.flops_per_forward(n_tok, n_kv)
    sec_block = flops_block / r["flops_per_s"]
    fps = FRAMES_PER_BLOCK_VIDEO / sec_block
    return {"value": fps, "unit": "FPS", "cores": r["cores"], "kind": "port",
            "sample": r["sample"] + f"; {r['flops_per_s'] / 1e9:.3f} GFLOP/s extrapolated linearly to "
                                    f"{flops_block / 1e12:.1f} TFLOP per block (extrapolated)",
            "sec_per_block_extrapolated": sec_block}


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port of its pinned
    matmul; the reference is Python and cannot travel to the GPU box) on all
    host cores.  A step is one bounded sample of the workload (~6 s of
    pinned-order matmul at the benchmark's token count, fewer seconds when K
    is large so the run stays within a few minutes); ``value`` extrapolates
    the measured rate to whole 14B blocks.  W warm-up samples of ~0.5 s.
    Rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    prof = profile_for(args.config)
    n_tok = 3 * prof.tokens_per_frame
    n_kv = prof.tokens_per_frame + 5 * n_tok
    k, w = max(1, args.steps), max(0, args.warmup)
    per = min(2.0, 40.0 / k)  # target seconds of matmul per sample (each sample's wall time is ~3x: process fan-out)
    for _ in range(w):
        cpu_baseline(prof, n_tok, n_kv, 4, target_s=0.5)
    vals, walls, cb = [], [], None
    for _ in range(k):
        t0 = time.perf_counter()
        cb = cpu_baseline(prof, n_tok, n_kv, 4, target_s=per)
        walls.append(time.perf_counter() - t0)
        vals.append(cb["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "FPS", "n_gpus": args.gpus,
            "steps": k, "warmup": w, "ms_per_step": 1e3 * statistics.mean(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": workload_config(args),
            "execution": {"executor": "reference CPU algorithm (oracle port of numerics.matmul), all host cores",
                          "step": "one bounded sample (pinned-order matmul at the block's token count); value = "
                                  "the sampled rate extrapolated linearly in FLOPs to whole blocks",
                          "sec_per_block_extrapolated": FRAMES_PER_BLOCK_VIDEO / v},
            "cpu_baseline": {"value": v, "unit": "FPS", "cores": cb["cores"], "kind": "port",
                             "sample": cb["sample"]},
            "e2e": {"value": v, "unit": "FPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "MEASURED_PEAKS.json"
    except OSError:
        return {}, None


def probe_kernels(stages, run_block, stream):
    """Eager per-kernel timing pass: CUDA events on the launch stream around
    every tagged kernel of one more block."""
    import torch

    evs = {}

    def probe(tag, phase, st):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(st or torch.cuda.current_stream())
        evs.setdefault(tag, []).append(ev)

    for st_ in stages:
        st_.eager = True
        st_.fw.probe = probe
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    run_block()
    p1.record(stream)
    torch.cuda.synchronize()
    for st_ in stages:
        st_.fw.probe = None
        st_.eager = False
    total = p0.elapsed_time(p1)
    kern = {}
    for tag, lst in evs.items():
        durs = [lst[2 * i].elapsed_time(lst[2 * i + 1]) for i in range(len(lst) // 2)]
        kern[tag] = {"launches": len(durs), "avg_ms": sum(durs) / len(durs), "sum_ms": sum(durs),
                     "share": sum(durs) / total}
    return kern, total


def roofline(prof, kern, n_tok, n_kv):
    """Roofline object for the dominant kernel (flash attention) plus the
    per-GEMM achieved TFLOP/s (algorithmic FLOPs / CUDA-event duration)."""
    # every kernel is timed inside a whole block of work (4 forwards, ~0.7 s of
    # back-to-back launches under the 1 kW power cap): the sustained peak is the
    # denominator (B200_PROFILING.md); the burst one is reported beside it
    peaks, src = _peaks()
    peak_tf = peaks.get("bf16_tflops_sustained", 1406.0)
    burst_tf = peaks.get("bf16_tflops", 1590.0)
    d, f = prof.model_dim, prof.ffn_dim
    flops = {"attention": 4.0 * n_tok * n_kv * d, "qkv": 2.0 * n_tok * d * 3 * d, "o_proj": 2.0 * n_tok * d * d,
             "ffn_up": 2.0 * n_tok * d * f, "ffn_down": 2.0 * n_tok * f * d}
    for tag, fl in flops.items():
        if tag in kern:
            kern[tag]["flops_per_launch"] = fl
            kern[tag]["tflops"] = fl / (kern[tag]["avg_ms"] / 1e3) / 1e12
            kern[tag]["frac_of_peak"] = kern[tag]["tflops"] / peak_tf
    # HBM-bound kernels: algorithmic bytes per launch / duration vs the measured copy bandwidth
    hbm = peaks.get("hbm_gbs", 6545.6)
    S = prof.tokens_per_frame
    eb = 2  # bf16 arena / activations
    bytes_ = {"norm_mod": n_tok * d * (4 + eb),                       # h fp32 in, xa bf16 out
              "sink_refresh": prof.n_layers * S * prof.n_heads * (prof.axes[0] // 2) * (8 + 2 * eb)
              + (prof.n_layers * S * prof.n_heads * 4 if prof.qk_norm else 0),  # temporal pairs: fp32 in, bf16 out
              "history_noise": (n_kv - S - n_tok) * d * (eb + eb)}     # ring rows in, scratch rows out (one of K/V)
    for tag, b in bytes_.items():
        if tag in kern:
            kern[tag]["bytes_per_launch"] = b
            kern[tag]["gbs"] = b / (kern[tag]["avg_ms"] / 1e3) / 1e9
            kern[tag]["frac_of_hbm"] = kern[tag]["gbs"] / hbm
    if "history_noise" in kern and os.environ.get("LP_HIST_OVERLAP", "0") == "1":
        kern["history_noise"]["note"] = ("side stream beside the GEMMs (lp_history_noise_co): the duration "
                                         "overlaps O-proj/FFN/QKV and is mostly off the critical path")
    if "attention" not in kern:
        return None
    ach = kern["attention"]["tflops"]
    return {"bound": "tensor", "kernel": "attn_tc2_kernel (cluster-pair tcgen05 flash attention + exact-rerun check + tail combine, one layer, all heads)",
            "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s", "frac": ach / peak_tf, "traffic": TRAFFIC.get(
                "attention"), "flops_per_launch": flops["attention"], "avg_launch_ms": kern["attention"]["avg_ms"],
            "share_of_step": kern["attention"]["share"], "frac_of_burst_peak": ach / burst_tf,
            "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside a whole block; burst "
                           f"{burst_tf} reported as frac_of_burst_peak)" if src else "fallback 1406 TFLOP/s"}


# dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed
# `ncu --set full` capture (profiles/); None until captured.
TRAFFIC = {}
try:
    TRAFFIC = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
except (OSError, ValueError):
    TRAFFIC = {}


def measure_decode(prof, latent, stream, dev, reps=10):
    """The decode stage on its own: one block's latent
    through the patch codec (VAE stand-in) to 12 pixel frames of 3 x 480 x 832
    fp32, timed with CUDA events; not part of the DiT step above."""
    import torch

    import paper_2512_04677_b200 as lp

    codec = lp.PatchVideoCodec(7, prof.channels, prof.height, prof.width, 3, 8, 4)
    dc = lp.DeviceCodec(codec, dev)
    out = torch.empty((latent.shape[0] * 4, codec.pixel_dim), device=f"cuda:{dev}")
    x = latent.contiguous()
    for _ in range(2):
        dc.decode_into(x, out, stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        dc.decode_into(x, out, stream)
    b.record(stream)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b) / reps
    nbytes = (x.numel() + out.numel()) * 4
    peaks, _ = _peaks()
    hbm = peaks.get("hbm_gbs", 6545.6)
    gbs = nbytes / (ms * 1e-3) / 1e9
    res = {"codec": "patch codec 16 -> 3 x 8 x 8 per latent location, r = 4 (the reference codec contract)",
           "frames_per_block": int(out.shape[0]), "ms_per_block": ms, "bytes_per_block": nbytes,
           "achieved_gbps": gbs, "frac_hbm": gbs / hbm}
    if prof.patched:  # the VAE stand-in: the decode GPU's realistic cost (vae.py)
        vae = lp.VaeDecoder(prof.channels, prof.height, prof.width, f"cuda:{dev}")
        for _ in range(2):
            vae.decode_into(x, out, stream)
        a.record(stream)
        for _ in range(3):
            vae.decode_into(x, out, stream)
        b.record(stream)
        torch.cuda.synchronize(dev)
        vms = a.elapsed_time(b) / 3
        fl = vae.flops_per_block()
        res["vae_stand_in"] = {
            "model": "Wan-2.1-VAE-like causal 3-D conv decoder, widths 384/384/192/128, 2 res blocks per stage, "
                     "implicit-GEMM tcgen05 convs (lp_conv_taps), random-init weights",
            "ms_per_block": vms, "tflop_per_block": fl / 1e12, "achieved_tflops": fl / (vms * 1e-3) / 1e12,
            "frac_of_dit_block": None}
        del vae
        torch.cuda.empty_cache()
    return res


def run_ours(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        return run_dist(args, rank, world, local)

    import paper_2512_04677_b200 as lp

    dev = local
    torch.cuda.set_device(dev)
    prof = profile_for(args.config)
    T, Lc = 4, 4
    cfg = lp.EngineConfig(mode="sequential", steps=T, cache_capacity=Lc, frames_per_block=3, profile=prof,
                          precision="bf16", devices=(dev,), device_inputs=True, blocks=1 << 20,
                          history_sigma=args.history_sigma)
    pipe = lp.StreamingPipeline(cfg)
    n_tok = 3 * prof.tokens_per_frame
    lat = prof.latent_dim
    K, W = args.steps, max(args.warmup, 3)
    total = W + K
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(11)
    noise_dev = torch.randn((total, 3, lat), generator=g, device=f"cuda:{dev}")
    # warm-up: block 0 (+ one-shot AAS), fill the rings, capture graphs
    for i in range(W):
        x = pipe.submit(i, noise_dev[i])
        if i == 0:
            torch.cuda.synchronize(dev)
            pipe.aas(x)
    pipe.capture()
    torch.cuda.synchronize(dev)
    n_kv_steady = prof.tokens_per_frame + Lc * n_tok + n_tok
    launches_per_block = pipe.kernels_per_block()

    # ---- value: device-resident inputs
    s = pipe.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        e0.record(s)
        for i in range(W, W + K):
            pipe.submit(i, noise_dev[i])
        e1.record(s)
        torch.cuda.synchronize(dev)
    dev_s = e0.elapsed_time(e1) / 1e3
    ms_step = 1e3 * dev_s / K
    fps = FRAMES_PER_BLOCK_VIDEO * K / dev_s

    # ---- e2e: pinned host noise in, latent out, through the streaming API
    host_in = torch.randn((K, 3, lat)).pin_memory()
    host_out = torch.empty((K, 3, lat)).pin_memory()
    base = W + K
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(s)
    for k in range(K):
        pipe.submit(base + k, host_in[k], out=host_out[k])
    e3.record(s)
    torch.cuda.synchronize(dev)
    e2e_s = e2.elapsed_time(e3) / 1e3
    wall_e2e = time.perf_counter() - t0
    e2e_fps = FRAMES_PER_BLOCK_VIDEO * K / e2e_s

    decode_stage = {} if args.no_decode else measure_decode(prof, noise_dev[0], s, dev)
    if decode_stage.get("vae_stand_in"):
        decode_stage["vae_stand_in"]["frac_of_dit_block"] = decode_stage["vae_stand_in"]["ms_per_block"] / ms_step

    kern, probe_ms = {}, None
    if not args.no_probe:
        kern, probe_ms = probe_kernels(list(pipe.stages.values()), lambda: pipe.submit(base + K, noise_dev[0]), s)
    roof = roofline(prof, kern, n_tok, n_kv_steady)
    peaks, _ = _peaks()
    peak_tf = peaks.get("bf16_tflops_sustained", 1406.0)
    burst_tf = peaks.get("bf16_tflops", 1590.0)
    flops_block = T * prof.flops_per_forward(n_tok, n_kv_steady)
    ach = flops_block * K / dev_s / 1e12
    line = {
        "metric": METRIC, "value": fps, "unit": "FPS", "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (device-RNG random-init weights, N(0,1) noise blocks)",
        "config": workload_config(args),
        "execution": {"parallelism": "1 GPU, T steps sequential (TPP stages collapsed)",
                   "block_latency_ms": ms_step, "achieved_tflops": ach, "frac_of_sustained_peak": ach / peak_tf,
                   "frac_of_burst_peak": ach / burst_tf,
                   "roofline_fps_sustained": FRAMES_PER_BLOCK_VIDEO / (flops_block / (peak_tf * 1e12)),
                   "roofline_fps_burst": FRAMES_PER_BLOCK_VIDEO / (flops_block / (burst_tf * 1e12)),
                   "frac_of_roofline_fps_sustained": fps / (FRAMES_PER_BLOCK_VIDEO / (flops_block / (peak_tf * 1e12))),
                   "ttff_ms_estimate": ms_step + decode_stage.get("ms_per_block", 0.0),
                   "ttff_note": "N=1, graphs captured: block 0 passes all T steps (one block latency) then the "
                                "decode stage; arrival offset 0",
                   "probe_block_ms": probe_ms},
        "e2e": {"value": e2e_fps, "unit": "FPS", "h2d_bytes_per_step": 3 * lat * 4,
                "d2h_bytes_per_step": 3 * lat * 4, "wall_s": wall_e2e},
        "gpu_launches": launches_per_block * K,
        "roofline": roof, "kernels": kern, "clocks": clk.summary(),
        "decode_stage": decode_stage,
    }
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(prof, n_tok, n_kv_steady, T)
        except Exception as exc:  # noqa: BLE001
            line["cpu_baseline"] = {"error": str(exc)}
    print(json.dumps(line), flush=True)


def run_dist(args, rank, world, local):
    """N > 1: one process per GPU, TPP stage groups (tpp_dist.DistTPP); each
    of the K timed steps advances the full pipeline(s) by one block, timed
    per rank with CUDA events on the rank's stream between barriers; the max
    over ranks is the job time."""
    import torch
    import torch.distributed as dist

    import paper_2512_04677_b200 as lp
    from paper_2512_04677_b200 import tpp_dist

    ndev = torch.cuda.device_count()
    local = local % ndev  # ranks may share a GPU (functional checks on a 1-GPU box)
    torch.cuda.set_device(local)
    if args.dist_backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        dist.init_process_group("gloo")
    prof = profile_for(args.config)
    T, Lc = 4, 4
    cfg = lp.EngineConfig(mode="tpp", steps=T, cache_capacity=Lc, frames_per_block=3, profile=prof,
                          precision="bf16", devices=(local,), device_inputs=True, blocks=1 << 20,
                          link_capacity=2, link_timeout_s=600.0, vae_decode=args.decode_gpu)
    run = tpp_dist.DistTPP(cfg, transport="ipc", device=local, decode_gpu=args.decode_gpu)
    role = run.role
    be = run.backend
    n_tok = 3 * prof.tokens_per_frame
    lat = prof.latent_dim
    K, W = args.steps, max(args.warmup, 3)
    # Staggered warm-up fills the pipeline: rank at position pos runs
    # W + (P - 1 - pos) blocks, so at the barrier every rank's next input is
    # already in its receive slot and each timed step is one block per stage
    # (steady streaming; the fill is a one-time stream start-up cost, TTFF).
    lead = len(role.ranks) - 1 - role.pos
    n_noise = W + len(role.ranks) + 2 * K + 2
    g = torch.Generator(device=f"cuda:{local}").manual_seed(11 + role.pipe)
    noise_dev = torch.randn((n_noise, 3, lat), generator=g, device=f"cuda:{local}")
    out_dev = torch.empty((3, lat), device=f"cuda:{local}")
    nxt = 0
    for i in range(W + lead):
        run.step(i, noise=noise_dev[i % n_noise], out=out_dev if i else None)
    nxt = W + lead
    run.finish()
    dist.barrier()
    torch.cuda.synchronize(local)
    n_kv_steady = prof.tokens_per_frame + Lc * n_tok + n_tok
    s = be.stream
    ends = []
    e0 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize(local)
        e0.record(s)
        for _ in range(K):
            run.step(nxt, noise=noise_dev[nxt % n_noise], out=out_dev)
            nxt += 1
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(s)
            ends.append(ev)
        torch.cuda.synchronize(local)
        run.finish()
        dist.barrier()
    el = e0.elapsed_time(ends[-1]) / 1e3
    dd = f"cuda:{local}" if args.dist_backend == "nccl" else "cpu"
    t = torch.tensor([el], dtype=torch.float64, device=dd)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    job_s = float(t.item())
    fps = FRAMES_PER_BLOCK_VIDEO * K * role.n_pipes / job_s
    steady = None
    if role.last and K >= 3:
        gaps = [ends[k - 1].elapsed_time(ends[k]) for k in range(1, K)]
        steady = FRAMES_PER_BLOCK_VIDEO / (statistics.median(gaps) / 1e3)

    # e2e: pinned host noise in on the first rank, pinned host latent out on the last
    host_in = torch.randn((K, 3, lat)).pin_memory()
    host_out = torch.empty((K, 3, lat)).pin_memory()
    dist.barrier()
    torch.cuda.synchronize(local)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(s)
    for k in range(K):
        run.step(nxt, noise=host_in[k], out=host_out[k])
        nxt += 1
    e3.record(s)
    torch.cuda.synchronize(local)
    run.finish()
    t = torch.tensor([e2.elapsed_time(e3) / 1e3], dtype=torch.float64, device=dd)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_fps = FRAMES_PER_BLOCK_VIDEO * K * role.n_pipes / float(t.item())

    kern = {}
    if not args.no_probe:
        kern, _ = probe_kernels(be.stages, lambda: run.step(nxt, noise=noise_dev[nxt % n_noise], out=out_dev), s)
        run.finish()
    roof = roofline(prof, kern, n_tok, n_kv_steady)
    steady_t = torch.tensor([steady or 0.0], dtype=torch.float64, device=dd)
    dist.all_reduce(steady_t, op=dist.ReduceOp.MAX)
    launches = torch.tensor([sum(st.fw.kernels_per_forward() for st in be.stages) * K], dtype=torch.int64,
                            device=dd)
    dist.all_reduce(launches)
    peaks, _ = _peaks()
    peak_tf = peaks.get("bf16_tflops_sustained", 1406.0)
    flops_block = T * prof.flops_per_forward(n_tok, n_kv_steady)
    if rank == 0:
        line = {
            "metric": METRIC, "value": fps, "unit": "FPS", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": 1e3 * job_s / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (device-RNG random-init weights, N(0,1) noise blocks)",
            "config": workload_config(args),
            "execution": {
                       "parallelism": f"TPP: {role.n_pipes} pipeline(s) x {len(role.ranks)} GPUs "
                                      f"(steps per GPU {[r.steps for r in run.roles[:len(role.ranks)]]}"
                                      f"{', last = decode rank' if args.decode_gpu else ''}), "
                                      "latents over NVLink P2P (CUDA IPC links, fused epilogue stores)",
                       "steady_fps_last_stage": float(steady_t.item()) * role.n_pipes,
                       "timed_region": "K pipeline steps (every stage one block) after a staggered "
                                       "warm-up that fills the pipeline; barrier-bracketed, max over ranks",
                       "achieved_tflops": flops_block * K * role.n_pipes / job_s / 1e12,
                       "roofline_fps_sustained": FRAMES_PER_BLOCK_VIDEO * min(len(role.ranks) - int(args.decode_gpu), T)
                       * role.n_pipes / (flops_block / (peak_tf * 1e12))},
            "e2e": {"value": e2e_fps, "unit": "FPS", "h2d_bytes_per_step": 3 * lat * 4 * role.n_pipes,
                    "d2h_bytes_per_step": 3 * lat * 4 * role.n_pipes},
            "gpu_launches": int(launches.item()),
            "roofline": roof, "kernels": kern, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    run.close()
    dist.barrier()
    dist.destroy_process_group()


def run_dropin(args):
    """FPS through the drop-in plug point the reference engine calls
    (Runtime.denoiser.denoise_block, engine.py:269-277), driven in the
    reference's run_sequential order (engine.py:255-285): per block and step
    a host latent in, a host velocity out, flow_step on the host, the
    KvEntry pushed into the reference-semantics RollingKvCache.  Every call
    synchronises (the plug-in contract returns numpy), so this is an
    end-to-end number by construction; timed by the host clock."""
    import numpy as np
    import torch

    import paper_2512_04677_b200 as lp
    from paper_2512_04677_b200.model import DeviceWeights

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    prof = profile_for(args.config)
    T, Lc = 4, 4
    sched = lp.TimestepSchedule.uniform(T)
    dw = DeviceWeights.random(prof, "bf16", f"cuda:{dev}", 7)
    dn = lp.B200Denoiser(None, sched, precision="bf16", device_weights=dw)
    K, W = args.steps, max(args.warmup, Lc + 1)
    conds = lp.synthetic_conditions(11, W + K, prof.audio_dim, prof.prompt_dim, prof.latent_dim)
    caches = {j: lp.RollingKvCache(j, Lc) for j in range(1, T + 1)}
    sink = lp.SinkSlot(conds.reference.copy(), 1)
    rng = np.random.default_rng(11)
    h2d = d2h = 0

    def block(i):
        nonlocal h2d, d2h
        x = lp.LatentBlock(rng.standard_normal((3, prof.latent_dim), dtype=np.float32), i)
        for j in range(T, 0, -1):
            o = dn.denoise_block(x, j, caches[j].view(), lp.BlockCond(conds.audio_for(i), conds.prompt),
                                 sink.content, i + 1, max_entries=Lc)
            h2d += x.values.nbytes
            d2h += o.velocity.nbytes
            x = lp.flow_step(x, o.velocity, sched.dt)
            caches[j].push(o.kv)
        return x

    for i in range(W):  # warm-up: fills the windows (steady N_kv from block L on)
        block(i)
    torch.cuda.synchronize(dev)
    h2d = d2h = 0
    with ClockSampler(dev) as clk:
        t0 = time.perf_counter()
        for i in range(W, W + K):
            block(i)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - t0
    fps = FRAMES_PER_BLOCK_VIDEO * K / wall
    line = {"metric": "streaming FPS through the drop-in denoise_block (reference engine loop order), 1 GPU",
            "value": fps, "unit": "FPS", "n_gpus": 1, "steps": K, "warmup": W, "ms_per_step": 1e3 * wall / K,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic latents/audio, random-init weights", "api": "dropin",
            "config": {"workload": workload(args.config), "path": "B200Denoiser.denoise_block x T per block, "
                       "host numpy latents, host flow_step, RollingKvCache window L=4 (N_kv 24,960 steady)"},
            "e2e": {"value": fps, "unit": "FPS", "h2d_bytes_per_step": h2d // K, "d2h_bytes_per_step": d2h // K,
                    "timer": "host perf_counter (every call synchronises)"},
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def run_long(args):
    """BASELINE config 4: a 14B-shape stream of ``--long-horizon`` blocks
    with RSFM (sink at i + delta, RoPE positions growing to N + 1, fp64
    angles), the rolling window and history noise, from a cold start:

    * TTFF = submit of block 0 -> its 12 frames decoded on the device,
      including the first (eager) forwards, the one-shot AAS sink swap and
      the graph capture that follows it (engine.py:255-285, PAPER.md TTFF);
    * whole-run FPS = 12 N / (stream start -> last block decoded);
      steady FPS over blocks > L (full window);
    * per-block latency from CUDA events on the pipeline stream;
    * drift = cosine similarity of every decoded frame with the decoded sink
      frame (metrics.drift_metric, engine.py:238), first vs last 10 %;
    * every block finite; the ring slots replayed against the reference
      window rule (RollingKvCache, kvcache.py:41-56) at every block."""
    import numpy as np
    import torch

    import paper_2512_04677_b200 as lp

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    prof = profile_for(args.config)
    T, Lc, N = 4, 4, args.long_horizon
    sigma = args.history_sigma
    cfg = lp.EngineConfig(mode="sequential", steps=T, cache_capacity=Lc, frames_per_block=3, profile=prof,
                          precision="bf16", devices=(dev,), device_inputs=True, blocks=N, history_sigma=sigma,
                          history_mode=args.history_mode)
    pipe = lp.StreamingPipeline(cfg)
    s = pipe.stream
    codec = lp.PatchVideoCodec(7, prof.channels, prof.height, prof.width, 3, 8, 4)
    dc = lp.DeviceCodec(codec, dev)
    lat = prof.latent_dim
    g = torch.Generator(device=f"cuda:{dev}").manual_seed(11)
    noise = torch.empty((3, lat), device=f"cuda:{dev}")
    frames = torch.empty((12, codec.pixel_dim), device=f"cuda:{dev}")
    drift = torch.empty((N, 12), device=f"cuda:{dev}")
    finite = torch.ones((), dtype=torch.bool, device=f"cuda:{dev}")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
    window = []  # reference replay: append, pop(0) beyond capacity

    def sink_frame():
        sk = torch.from_numpy(np.asarray(pipe.sink.content, np.float32)).to(f"cuda:{dev}").reshape(1, lat)
        out = torch.empty((4, codec.pixel_dim), device=f"cuda:{dev}")
        dc.decode_into(sk, out, s)
        return out[0]

    def one(i, ref):
        with torch.cuda.stream(s):
            noise.normal_(generator=g)
        ev[i][0].record(s)
        x = pipe.submit(i, noise)
        with torch.cuda.stream(s):
            dc.decode_into(x.reshape(3, lat), frames, s)
            drift[i] = (frames @ ref) / (frames.norm(dim=1) * ref.norm())
            finite.logical_and_(torch.isfinite(x).all())
        ev[i][1].record(s)
        window.append(i)
        if len(window) > Lc:
            window.pop(0)
        for st in pipe.stages.values():
            if st.ring.blocks != window:
                raise AssertionError(f"ring replay diverged at block {i}: {st.ring.blocks} vs {window}")
        return x

    torch.cuda.synchronize(dev)
    with ClockSampler(dev) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_start.record(s)
        x0 = one(0, sink_frame())
        pipe.aas(x0)  # host round trip: part of the first-block bubble
        ref = sink_frame()  # drift reference: the swapped sink
        pipe.capture()
        t_first = torch.cuda.Event(enable_timing=True)
        t_first.record(s)
        for i in range(1, N):
            one(i, ref)
        t_end = torch.cuda.Event(enable_timing=True)
        t_end.record(s)
        torch.cuda.synchronize(dev)
    total_s = t_start.elapsed_time(t_end) / 1e3
    ttff_ms = t_start.elapsed_time(t_first)
    lat_ms = np.array([a.elapsed_time(b) for a, b in ev])
    steady = lat_ms[Lc + 1:] if N > Lc + 2 else lat_ms[1:]
    d = drift.float().cpu().numpy()
    k = max(1, N // 10)
    line = {"metric": "long-horizon stream (BASELINE config 4): whole-run FPS", "value": 12 * N / total_s,
            "unit": "FPS", "n_gpus": 1, "steps": N, "warmup": 0, "ms_per_step": 1e3 * total_s / N,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic noise (device Philox), random-init weights", "api": "stream",
            "config": {"workload": workload(args.config) + f", {N} blocks = {12 * N} video frames from a cold start",
                       "history_sigma": sigma, "history_mode": args.history_mode, "window": Lc,
                       "sink_positions": [1 + 1, N + 1]},
            "fps_steady": 12e3 / float(np.mean(steady)), "ttff_ms": ttff_ms,
            "ttff_note": "block 0 (eager) + decode + AAS sink swap + graph capture",
            "block_ms": {"p50": float(np.percentile(steady, 50)), "p99": float(np.percentile(steady, 99)),
                         "max": float(steady.max())},
            "drift": {"first_10pct_mean": float(d[:k].mean()), "last_10pct_mean": float(d[-k:].mean()),
                      "min": float(d.min()), "finite": bool(np.isfinite(d).all())},
            "all_blocks_finite": bool(finite.item()), "ring_replay": "ok",
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.long_horizon:
        run_long(args)
        return
    if args.impl == "reference":
        run_reference(args)
    elif args.api == "dropin":
        run_dropin(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
