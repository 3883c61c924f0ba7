#!/usr/bin/env python3
"""Benchmark of the B200 binarized-CNN forward pass (arXiv 1808.00209) -- the driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl bnn|reference] [--total-batch B] [--mode rgb]
    torchrun --nproc-per-node N bench.py --gpus N ...

A "step" is one pass of the whole hot path (bnn_forward: conv1 (+ fused input binarization, threshold,
pool) -> conv2 + pool -> FC1 -> FC2 -> FC3 + argmax) over BASELINE config 5's batch: 262,144 synthetic
images per step, split into contiguous shards over the N GPUs (strong scaling; --batch B instead fixes
B images per GPU = weak scaling), followed at N > 1 by the NCCL all-gather of the predictions.  Inputs are
resident in HBM before the timed region; the 7.25 GB input (906 MB per GPU at N = 8) is larger than the
126 MB L2, so no L2 flush is needed.

Prints ONE JSON line (rank 0).  `value` = images/s of the whole job, timed with CUDA events on the
forward stream, max over ranks.  `e2e` = the same metric through bnn_forward_host (pinned host images
-> host logits/classes, copies inside the timed region).  `roofline` = the dominant conv kernel
(largest live CUDA-event time): tcgen05 kernels as TOPS (2 x algorithmic binary MACs / time) vs the
measured bf16 peak x the nominal ratio of the kernel's operand type (burst when the SM clock held its
maximum during the timed region, else sustained), plus the repo's probed MMA rate; POPC kernels as
algorithmic popcounts / time vs the POPC pipe (16 / clk / SM, tools/probes/pipe_probe.cu).
`parity` = sampled images of the whole job vs the CPU oracle; `multi_gpu_check` (N > 1) = the gathered
predictions vs a 1-GPU pass over the same global batch on rank 0.
`cpu_baseline` = the CPU oracle (oracle/) on a bounded sample on the host cores (rank 0, N = 1).
--impl reference times that oracle alone as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "images/sec at 1/2/4/8 B200; binary conv popc-pipe % and HBM GB/s (ncu)"
POPC_PER_CLK_SM = 16  # measured on B200: profiles/pipe_probe_r01.txt
MODES = {"rgb": 1, "gray": 2, "lbp": 3, "none": -1, "sign": 0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="bnn", choices=["bnn", "reference"])
    ap.add_argument("--total-batch", type=int, default=262144,
                    help="images per step over all GPUs (BASELINE config 5; strong scaling, contiguous shards)")
    ap.add_argument("--batch", type=int, default=0, help="if set: fixed images per GPU per step (weak scaling)")
    ap.add_argument("--chunk", type=int, default=65536, help="bnn_net max_batch (images per internal chunk; 65536 measured best at 262144 images per step: 14.2-14.4 vs 14.2 M img/s for 16384, tools/ab_chunks.sh)")
    ap.add_argument("--mode", default="rgb", choices=sorted(MODES))
    ap.add_argument("--seed", type=int, default=2018)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--check", type=int, default=8, help="sampled images checked against the oracle after timing")
    ap.add_argument("--opt", action="append", default=[], metavar="KEY=V",
                    help="bnn_set_option before the run (A/B of kernel variants; results are identical for every setting)")
    ap.add_argument("--config", default="vehicle", choices=["vehicle", "latency", "modes", "cifar", "sweep", "alg1"],
                    help="vehicle = the headline (default); latency = BASELINE config 1 (batch 1, 1000 images); "
                         "modes = config 2 (batch 4096, every input binarization); cifar = config 4; "
                         "sweep = config 3 (single binary conv layers)")
    return ap.parse_args()


# ----------------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.file = None

    def start(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", delete=False, suffix=".csv")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.file,
                                         stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.file.flush()
        rows = [ln.split(",") for ln in open(self.file.name).read().strip().splitlines() if ln.strip()]
        os.unlink(self.file.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 7:
                continue
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for nm, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def conv_popc_per_image(spec, mode):
    """Algorithmic popcounts per image and per conv layer: H*W*C_out*K^2*ceil(C_in/32),
    dense patch (ceil(K^2 C_in / 32) words) for the first layer with C_in < 32."""
    from paper_1808_00209_b200 import synth
    h, w, c = spec["h"], spec["w"], synth.input_channels(spec["c"], mode)
    out, macs = [], []
    for L in spec["layers"]:
        if L["kind"] == "conv":
            k, co = L["k"], L["c_out"]
            words = -(-k * k * c // 32) if c < 32 else k * k * (-(-c // 32))
            out.append(h * w * co * words)
            macs.append(h * w * co * k * k * c)
            c = co
            h //= L.get("pool", 1)
            w //= L.get("pool", 1)
        else:
            d = h * w * c
            out.append(L["l"] * (-(-d // 32)))
            macs.append(L["l"] * d)
            h, w, c = 1, 1, L["l"]
    return out, macs


def oracle_sample(spec, mode, seconds: float, threads: int, seed: int):
    """Time the CPU oracle (as it stands) on about `seconds` of work: images/s and images done."""
    import numpy as np
    from oracle import oracle as orc
    from paper_1808_00209_b200 import synth
    layers = synth.make_weights(spec, mode, seed)
    T = synth.thresholds(3, seed).numpy() if mode == 1 else (np.array([-127.0], np.float32) if mode == 2 else None)
    om = {0: orc.SIGN, 1: orc.THRESH_RGB, 2: orc.THRESH_GRAY, 3: orc.LBP, -1: orc.NONE}[mode]
    net = orc.Net(spec["h"], spec["w"], spec["c"], om, T, [dict(L, wt=L["wt"].numpy()) for L in layers])
    imgs = synth.images(threads, spec["h"], spec["w"], spec["c"], seed + 1).numpy()
    done, t0 = 0, time.perf_counter()
    while True:
        net.forward(imgs, threads=threads)
        done += threads
        el = time.perf_counter() - t0
        if el >= seconds:
            return done / el, done, el


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1



def read_peaks():
    """MEASURED_PEAKS.json (driver-written) else the B200_PROFILING.md fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return {"hbm_gbs": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sustained": d.get("bf16_tflops_sustained",
                    d["bf16_tflops"]), "source": "measured (MEASURED_PEAKS.json)"}
        except (ValueError, KeyError):
            pass
    return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "source": "fallback (B200_PROFILING.md)"}


# tcgen05 MMA rates measured by the repo's probes (M = 128, N >= 128, 148 CTAs): MAC / clk / SM
PROBE_MAC_PER_CLK_SM = {"i8": 8187, "fp4": 16375}  # profiles/umma_probe_r01.txt, profiles/mxf4_probe_r01.txt


def kernel_dtype(kernel: str):
    """Operand type of a kernel family: 'fp4' (tcgen05 kind::mxf4), 'i8' (kind::i8) or None (integer pipe)."""
    if "tc4" in kernel or "fp4" in kernel:
        return "fp4"
    if "_tc" in kernel or "_tma_" in kernel:
        return "i8"
    return None


def clocks_held(clocks) -> bool:
    """True when the SM clock stayed at its maximum with no throttle reason during the timed region:
    the kernel then runs at the burst (not the sustained, power-limited) tensor rate."""
    sm, mx = clocks.get("sm_mhz"), clocks.get("sm_max_mhz")
    return bool(sm and mx and sm >= 0.97 * mx and not clocks.get("reasons"))


def tensor_peak(dt: str, clocks, sms: int):
    """Peak dense TOPS (2 ops per MAC) for operand type dt: the measured bf16 peak of MEASURED_PEAKS.json x the
    nominal ratio (i8 2x, fp4 4x; B200_PROFILING.md), burst when the clocks held (clocks_held) else sustained;
    plus the MMA rate the repo's own probes measured x SMs x the median SM clock under load."""
    peaks = read_peaks()
    ratio = 4.0 if dt == "fp4" else 2.0
    burst, sustained = ratio * peaks["bf16"], ratio * peaks["bf16_sustained"]
    held = clocks_held(clocks)
    mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    probe = 2.0 * PROBE_MAC_PER_CLK_SM[dt] * sms * mhz * 1e6 / 1e12
    return {"peak": burst if held else sustained, "peak_burst": burst, "peak_sustained": sustained,
            "peak_probe": probe,
            "peak_basis": "%s dense = %g x bf16 %s %.1f TFLOP/s, %s; %s" % (
                dt, ratio, "burst" if held else "sustained", peaks["bf16"] if held else peaks["bf16_sustained"],
                peaks["source"], "SM clock held at max with no throttle reason during the timed region -> burst"
                if held else "SM clock below max or throttled during the timed region -> sustained"),
            "peak_probe_basis": "tcgen05 %s probe %d MAC/clk/SM x %d SMs x %.0f MHz (median under load) x 2" % (
                dt, PROBE_MAC_PER_CLK_SM[dt], sms, mhz)}


def roofline_for(kernel: str, macs: float, popc: float, ms: float, clocks, sms: int):
    """Roofline of one kernel: `macs` algorithmic binary MACs (and `popc` popcounts) per launch in `ms`."""
    dt = kernel_dtype(kernel)
    sm_max = clocks.get("sm_max_mhz") or 1965.0
    popc_peak = POPC_PER_CLK_SM * sms * sm_max * 1e6
    if dt is not None:
        achieved = 2.0 * macs / (ms * 1e-3) / 1e12
        p = tensor_peak(dt, clocks, sms)
        r = {"bound": "tensor", "pipe": "tcgen05 kind::%s" % ("mxf4" if dt == "fp4" else "i8"),
             "unit": "TOPS (%s, 2 x binary MAC)" % ("fp4" if dt == "fp4" else "int8"), "achieved": achieved}
        r.update(p)
        r["frac"] = achieved / p["peak"]
        r["frac_burst"] = achieved / p["peak_burst"]
        r["frac_sustained"] = achieved / p["peak_sustained"]
        r["frac_probe"] = achieved / p["peak_probe"]
        r["popc_equivalent_frac"] = popc / (ms * 1e-3) / popc_peak
    else:
        achieved = popc / (ms * 1e-3) / 1e12
        r = {"bound": "alu", "pipe": "POPC (16/clk/SM, measured: profiles/pipe_probe_r01.txt)", "unit": "Tpopc/s",
             "achieved": achieved, "peak": popc_peak / 1e12,
             "peak_basis": "16 POPC/clk/SM x %d SMs x %.0f MHz (sm max clock)" % (sms, sm_max)}
        r["frac"] = achieved / r["peak"]
    return r


def dominant_roofline(net, spec, mode, stage_ms, stage_launch, images_total, clocks, dev):
    """Roofline object for the conv layer with the largest live CUDA-event time (roofline_for)."""
    import torch
    popc_img, mac_img = conv_popc_per_image(spec, mode)
    conv_stages = [i for i, Ly in enumerate(spec["layers"]) if Ly["kind"] == "conv"]
    dom = max(conv_stages, key=lambda i: stage_ms[i + 1])
    launches = max(1, stage_launch[dom + 1])
    ms_per_launch = stage_ms[dom + 1] / launches
    imgs_per_launch = images_total / launches
    kernel = net.layer_kernel(dom, int(imgs_per_launch))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    r = roofline_for(kernel, mac_img[dom] * imgs_per_launch, popc_img[dom] * imgs_per_launch, ms_per_launch, clocks, sms)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile)).get("layer%d" % dom)
            if tj and kernel in tj["kernel"]:
                traffic = tj["dram_bytes_per_launch"] * imgs_per_launch / tj["images_per_launch"]
        except (ValueError, KeyError):
            traffic = None
    step_ms = sum(stage_ms)
    r.update({"kernel": "layer%d %s" % (dom, kernel), "traffic": traffic, "ms_per_launch": ms_per_launch,
              "images_per_launch": imgs_per_launch,
              "algorithmic": "%d binary MAC x 2 ops per image x %d images per launch" % (mac_img[dom], imgs_per_launch),
              "kernel_share_of_step": stage_ms[dom + 1] / step_ms if step_ms else None})
    return r

# ----------------------------------------------------------------------------------- reference arm
def run_reference(a, rank, world):
    """The reference arm: the CPU oracle on the host cores, same metric/config, each step a bounded
    sample (one image per core).  Under torchrun only rank 0 works."""
    if rank != 0:
        return
    from paper_1808_00209_b200 import synth
    spec = synth.VEHICLE
    mode = MODES[a.mode]
    cores = host_cores()
    for _ in range(a.warmup):
        oracle_sample(spec, mode, 0.0, cores, a.seed)
    t0 = time.perf_counter()
    n = 0
    for _ in range(a.steps):
        _, d, _ = oracle_sample(spec, mode, 0.0, cores, a.seed)
        n += d
    el = time.perf_counter() - t0
    v = n / el
    line = {"metric": METRIC, "value": v, "unit": "images/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": el * 1e3 / a.steps, "higher_is_better": True,
            "scaling": "weak" if a.batch else "strong", "vs_baseline": None,
            "dtype": "i64", "data": "synthetic", "impl": "reference",
            "config": {"workload": "vehicle classifier (PAPER.md Table 2: conv32x5x5+pool, conv32x5x5+pool, FC100, "
                                   "FC100, FC4), %s input binarization, %d images per step (BASELINE config 5); each "
                                   "timed step is a bounded sample of %d of them (one per host core)" % (
                                       a.mode, a.batch * world if a.batch else a.total_batch, cores),
                       "batch_per_step": cores},
            "cpu_baseline": {"value": v, "unit": "images/s", "cores": cores, "cpu_model": cpu_model(), "kind": "oracle",
                             "sample": "%d steps x %d images (vehicle net, %s)" % (a.steps, cores, a.mode)},
            "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------- bnn arm
def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def workload(a, world):
    """(start, n, n_max, total, scaling) of this rank: strong scaling over --total-batch (BASELINE config 5,
    contiguous shards, dist.shard_total) unless --batch sets a fixed per-GPU batch (weak scaling)."""
    from paper_1808_00209_b200 import dist as bdist
    rank = int(os.environ.get("RANK", "0"))
    if a.batch:
        start, n = bdist.shard(a.batch, rank)
        return start, n, a.batch, a.batch * world, "weak"
    start, n = bdist.shard_total(a.total_batch, rank, world)
    return start, n, -(-a.total_batch // world), a.total_batch, "strong"


def assemble_predictions(logits_all, cls_all, total, world, n_max, scaling):
    """Global-order predictions from the padded all-gather buffers ([world * n_max, ...], rank r's shard
    in rows [r * n_max, r * n_max + size_r))."""
    import torch
    from paper_1808_00209_b200 import dist as bdist
    sizes = [bdist.shard_total(total, r, world)[1] if scaling == "strong" else n_max for r in range(world)]
    return (torch.cat([logits_all[r * n_max:r * n_max + sizes[r]] for r in range(world)]),
            torch.cat([cls_all[r * n_max:r * n_max + sizes[r]] for r in range(world)]))


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return run_reference(a, rank, world)
    if a.opt:
        import paper_1808_00209_b200 as bnn
        for kv in a.opt:
            k, v = kv.split("=")
            bnn.set_option(k, int(v))
    if a.config != "vehicle":
        return {"latency": run_latency, "modes": run_modes, "cifar": run_cifar, "sweep": run_sweep,
                "alg1": run_alg1}[a.config](a)

    import torch
    import torch.distributed as dist
    import paper_1808_00209_b200 as bnn
    from paper_1808_00209_b200 import dist as bdist
    from paper_1808_00209_b200 import synth

    assert torch.cuda.is_available(), "bench.py needs a GPU (the CUDA path has no CPU fallback)"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    spec = synth.VEHICLE
    mode = MODES[a.mode]
    start, B, n_max, total, scaling = workload(a, world)

    # weights: identical on every rank (same seed), packed on the device by bnn_pack(SIGN)
    layers = synth.make_weights(spec, mode, a.seed)
    dl = [dict(L, wt=bnn.pack_weights(L["wt"].to(dev))) for L in layers]
    T = None
    if mode == 1:
        T = synth.thresholds(3, a.seed).to(dev)
    elif mode == 2:
        T = torch.tensor([-127.0], device=dev)
    net = bnn.Net(spec["h"], spec["w"], spec["c"], bnn.U8, mode, T, dl, max_batch=min(a.chunk, B))
    # this rank's contiguous shard of the seeded stream (4096-image chunks: identical data for any N)
    images = synth.images_chunked(start, B, spec["h"], spec["w"], spec["c"], a.seed + 1, device=dev)
    L = spec["layers"][-1]["l"]
    # prediction buffers padded to the largest shard so the all-gather has equal sizes
    logits_pad = torch.zeros((n_max, L), dtype=torch.int32, device=dev)
    cls_pad = torch.full((n_max,), -1, dtype=torch.int32, device=dev)
    logits, cls = logits_pad[:B], cls_pad[:B]
    if world > 1:
        logits_all = torch.empty((world * n_max, L), dtype=torch.int32, device=dev)
        cls_all = torch.empty((world * n_max,), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        net.forward(images, logits, cls)
        if world > 1:
            bdist.gather_predictions(logits_pad, cls_pad, logits_all, cls_all)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / a.steps
    clocks["timed_region_s"] = round(ms * a.steps / 1e3, 3)
    ms = bdist.max_over_ranks(ms, dev)
    value = total / (ms * 1e-3)
    # per-stage live kernel times: the same steps again with the library's CUDA events around every
    # launch (kept out of the timed region: events between kernels serialise programmatic launches)
    bnn.set_option("streams", 1)  # one stream here, so a kernel's event time is its own duration
    net.forward(images, logits, cls)  # warm (first-launch costs stay out of the per-stage times)
    torch.cuda.synchronize()
    prof_steps = max(1, min(a.steps, 5))
    net.profile(True)
    for _ in range(prof_steps):
        net.forward(images, logits, cls)
    torch.cuda.synchronize()
    stage_ms, stage_launch = net.profile_read()
    net.profile(False)
    bnn.set_option("streams", 2)

    # ---- roofline of the dominant conv kernel (live CUDA-event times of its launches)
    roofline = dominant_roofline(net, spec, mode, stage_ms, stage_launch, B * prof_steps, clocks, dev)
    stages = {("pack" if i == 0 else ("layer%d" % (i - 1) if i <= len(spec["layers"]) else "argmax")):
              round(stage_ms[i] / prof_steps, 4) for i in range(len(stage_ms)) if stage_launch[i]}

    # ---- end to end through bnn_forward_host (pinned host in, host out)
    e2e = None
    if not a.no_e2e:
        h_images = torch.empty(images.shape, dtype=torch.uint8, pin_memory=True)
        h_images.copy_(images)
        h_logits = torch.empty((B, L), dtype=torch.int32, pin_memory=True)
        h_cls = torch.empty((B,), dtype=torch.int32, pin_memory=True)
        ke = max(3, min(a.steps, 5))
        net.forward_host(h_images, h_logits, h_cls)  # warm the staging buffers
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ke):
            net.forward_host(h_images, h_logits, h_cls)
        el = bdist.max_over_ranks((time.perf_counter() - t0) / ke, dev)
        assert torch.equal(h_cls, cls.cpu()), "forward_host disagrees with forward"
        e2e = {"value": total / el, "unit": "images/s", "h2d_bytes_per_step": int(h_images.numel()) * world,
               "d2h_bytes_per_step": int(h_logits.numel() * 4 + h_cls.numel() * 4) * world, "steps": ke,
               "timing": "wall clock around the synchronous C-ABI call (pinned host images in, host logits/classes "
                         "out), max over ranks"}
        del h_images

    # ---- predictions of the whole job, in global image order (rank 0)
    parity, multi = None, None
    if world > 1:
        g_logits, g_cls = assemble_predictions(logits_all, cls_all, total, world, n_max, scaling)
    else:
        g_logits, g_cls = logits, cls
    if rank == 0 and world > 1:
        # the gathered N-GPU predictions must be bit-identical to a 1-GPU pass over the same global batch
        # (the images are independent, SURVEY row e); rank 0 regenerates the whole batch and runs it alone
        del images
        torch.cuda.empty_cache()
        full = synth.images_chunked(0, total, spec["h"], spec["w"], spec["c"], a.seed + 1, device=dev)
        ref_l, ref_c = net.forward(full)
        ok = bool(torch.equal(ref_l, g_logits) and torch.equal(ref_c, g_cls))
        multi = {"images": total, "gathered_equals_1gpu_pass": ok}
        del full
        assert ok, "gathered %d-GPU predictions differ from the 1-GPU pass" % world
    if a.check > 0 and rank == 0:
        # sampled images spread over the WHOLE job (every shard, incl. the last image) against the oracle
        import numpy as np
        from oracle import oracle as orc
        idx = np.unique(np.linspace(0, total - 1, a.check).astype(int))
        om = {0: orc.SIGN, 1: orc.THRESH_RGB, 2: orc.THRESH_GRAY, 3: orc.LBP, -1: orc.NONE}[mode]
        onet = orc.Net(spec["h"], spec["w"], spec["c"], om, None if T is None else T.cpu().numpy(),
                       [dict(Ly, wt=Ly["wt"].numpy()) for Ly in layers])
        # regenerated from the seeded stream on the device (the CUDA generator's stream, as the timed inputs)
        sample = torch.cat([synth.images_chunked(int(i), 1, spec["h"], spec["w"], spec["c"], a.seed + 1, device=dev)
                            for i in idx]).cpu().numpy()
        ref_l, ref_c = onet.forward(sample, threads=min(len(idx), host_cores()))
        ok = bool(np.array_equal(g_logits[idx].cpu().numpy(), ref_l) and np.array_equal(g_cls[idx].cpu().numpy(), ref_c))
        parity = {"images_checked": int(len(idx)), "global_indices": [int(i) for i in idx], "bit_exact": ok}
        assert ok, "sampled parity against the oracle FAILED"

    cpu = None
    if not a.no_cpu and rank == 0 and world == 1:
        cores = host_cores()
        v, done, el = oracle_sample(spec, mode, 12.0, cores, a.seed)
        cpu = {"value": v, "unit": "images/s", "cores": cores, "cpu_model": cpu_model(), "kind": "oracle",
               "sample": "%d vehicle images (%s), %.1f s on %d threads, one image per thread" % (done, a.mode, el, cores)}

    launches = bnn.forward_launches(net, B) * a.steps
    _, mac_img = conv_popc_per_image(spec, mode)
    tot_mac = sum(mac_img) * total
    line = {"metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": {"workload": "vehicle classifier (PAPER.md Table 2: conv32x5x5+pool, conv32x5x5+pool, FC100, "
                                   "FC100, FC4), %s input binarization, %d images per step over %d GPU(s)%s" % (
                                       a.mode, total, world, " (BASELINE config 5)" if total == 262144 else ""),
                       "global_batch": total, "batch_per_gpu": B, "chunk": min(a.chunk, B),
                       "input": "u8 96x96x3 uniform, resident in HBM",
                       "l2": "inputs (%d MB/GPU) larger than L2; no flush" % (B * 27648 // 2 ** 20),
                       "parallelism": "dp%d (contiguous shards; NCCL all-gather of predictions)" % world},
            "binary_mac_per_s": tot_mac / (ms * 1e-3), "stage_ms_per_step": stages,
            "roofline": roofline, "clocks": clocks, "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu,
            "parity": parity, "multi_gpu_check": multi}
    if a.opt:
        line["config"]["options"] = a.opt
    if rank == 0:
        print(json.dumps(line), flush=True)
    net.close()
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------------- extra configs
def _net_for(spec, mode, seed, dev, max_batch):
    import torch
    import paper_1808_00209_b200 as bnn
    from paper_1808_00209_b200 import synth
    layers = synth.make_weights(spec, mode, seed)
    dl = [dict(L, wt=bnn.pack_weights(L["wt"].to(dev))) for L in layers]
    T = synth.thresholds(3, seed).to(dev) if mode == 1 else (
        torch.tensor([-127.0], device=dev) if mode == 2 else None)
    return bnn.Net(spec["h"], spec["w"], spec["c"], bnn.U8, mode, T, dl, max_batch=max_batch), layers, T


def _timed(fn, steps, warmup, min_s: float = 0.0):
    """ms per call of fn over `steps` calls (more if needed to fill min_s seconds), after `warmup` calls."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if min_s > 0:
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        steps = max(steps, int(min_s * 1e3 / max(e0.elapsed_time(e1), 1e-3)) + 1)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def _timed_clocks(fn, steps, warmup, min_s: float = 0.5):
    """_timed with the nvidia-smi clock sampler running over the timed region: (ms, clocks)."""
    import torch
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    time.sleep(0.25)
    ms = _timed(fn, steps, warmup, min_s)
    clocks = sampler.stop()
    return ms, clocks


def _emit(d):
    print(json.dumps(d), flush=True)


def run_latency(a):
    """BASELINE config 1 / the paper's protocol: 1000 random images fed one at a
    time; the timer starts after the image is on the device and stops after the last kernel.  Here
    one image = one CUDA-graph replay (bnn_forward_staged), timed with an event pair per image."""
    import torch
    import paper_1808_00209_b200 as bnn
    from paper_1808_00209_b200 import synth
    dev = torch.device("cuda", 0)
    net, _, _ = _net_for(synth.VEHICLE, 1, a.seed, dev, 64)
    st_in, st_lg, st_cls = net.staging(1)
    imgs = synth.images(1000, 96, 96, 3, a.seed + 1, device=dev)
    for i in range(10):
        st_in.copy_(imgs[i:i + 1])
        net.forward_staged(1)
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    sampler.start()
    time.sleep(0.25)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(1000)]
    for i in range(1000):
        st_in.copy_(imgs[i:i + 1])  # the "memory copy" of the paper's protocol, outside the timer
        ev[i][0].record()
        net.forward_staged(1)
        ev[i][1].record()
    torch.cuda.synchronize()
    per = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
    b2b = _timed(lambda: net.forward_staged(1), 1000, 20, 0.3) * 1e3
    device = _device_latency(bnn, synth, dev, imgs[:200])
    clocks = sampler.stop()
    _emit({"metric": "latency per image, batch 1 (kernel time)", "value": sum(per) / len(per), "unit": "us",
           "higher_is_better": False, "median_us": per[len(per) // 2], "p99_us": per[int(0.99 * len(per))],
           "back_to_back_us": b2b, "images_per_s_back_to_back": 1e6 / b2b,
           "device_us_per_image": device,
           "note": "value / back_to_back: one graph replay per image, bound by the host's cudaGraphLaunch (~16 us); "
                   "device_us_per_image: 200 single-image forwards captured in one CUDA graph (launch cost amortised), "
                   "for the default whole-network cluster kernel (f1; the default for chunks of <= 12 images) and the 5-kernel PDL path",
           "config": {"workload": "config 1: vehicle classifier, THRESH_RGB, 1000 random images one at a time, "
                                  "one CUDA graph replay per image",
                      "kernel": "fused_cluster_kernel" if bnn.forward_launches(net, 1) == 1 else net.layer_kernel(0, 1)},
           "context": "paper: 55.63 us per image on a GTX 1080 (Table 1, PAPER.md:292)",
           "gpu_launches_per_image": bnn.forward_launches(net, 1), "clocks": clocks})


def _device_latency(bnn, synth, dev, imgs):
    """Device-side batch-1 latency (us per image) of the whole-network cluster kernel (f1, the default for one image)
    and of the 5-kernel PDL path: len(imgs) single-image forwards captured back to back in ONE CUDA graph, so the
    host launch cost is paid once per graph; the two paths' classes must agree."""
    import torch
    R = imgs.shape[0]
    out = {}
    classes = []
    for name, fused in (("fused_cluster", 1), ("pdl_graph", 0)):
        bnn.set_option("fused_max_n", fused)
        net, _, _ = _net_for(synth.VEHICLE, 1, 2018, dev, 8)
        lg = torch.empty((R, 4), dtype=torch.int32, device=dev)
        cls = torch.empty((R * 4,), dtype=torch.int32, device=dev)  # image i's class at 4 i (16-byte aligned)
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            for i in range(3):
                net.forward(imgs[i:i + 1], lg[i:i + 1], cls[4 * i:4 * i + 1])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(R):
                net.forward(imgs[i:i + 1], lg[i:i + 1], cls[4 * i:4 * i + 1])
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) * 1e3 / (10 * R)
        classes.append(cls[::4].clone())
        net.close()
    bnn.set_option("fused_max_n", 12)  # (the default)
    out["classes_identical"] = bool(torch.equal(classes[0], classes[1]))
    out["images_per_graph"] = R
    return out


def _stage_profile(net, fn, reps=3):
    """Per-stage live times (ms per call) of fn on one stream, AFTER a warm call (first-launch costs excluded)."""
    import torch
    import paper_1808_00209_b200 as bnn
    bnn.set_option("streams", 1)
    fn()
    torch.cuda.synchronize()
    net.profile(True)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    sms, cnt = net.profile_read()
    net.profile(False)
    bnn.set_option("streams", 2)
    return [x / reps for x in sms], [c // reps for c in cnt]


def _layer_rooflines(net, spec, mode, stage_ms, stage_cnt, B, clocks):
    """roofline_for of every conv / dense layer of a net run over B images (live per-stage times)."""
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    popc, macs = conv_popc_per_image(spec, mode)
    out = []
    for i in range(len(spec["layers"])):
        t, c = stage_ms[i + 1], max(1, stage_cnt[i + 1])
        if t <= 0:
            continue
        kernel = net.layer_kernel(i, B // c if c > 1 else B)
        r = roofline_for(kernel, macs[i] * B / c, popc[i] * B / c, t / c, clocks, sms)
        out.append({"layer": i, "kernel": kernel, "ms": round(t, 4), "bound": r["bound"], "unit": r["unit"],
                    "achieved": round(r["achieved"], 1), "peak": round(r["peak"], 1), "frac": round(r["frac"], 4),
                    **({"frac_probe": round(r["frac_probe"], 4)} if "frac_probe" in r else {})})
    return out


def run_modes(a):
    """BASELINE config 2: batch 4096 on one B200 for every input-binarization variant."""
    import torch
    from paper_1808_00209_b200 import synth
    dev = torch.device("cuda", 0)
    B = 4096
    imgs = synth.images(B, 96, 96, 3, a.seed + 1, device=dev)
    for name in ["rgb", "gray", "lbp", "none", "sign"]:
        mode = MODES[name]
        net, _, _ = _net_for(synth.VEHICLE, mode, a.seed, dev, B)
        lg = torch.empty((B, 4), dtype=torch.int32, device=dev)
        cls = torch.empty((B,), dtype=torch.int32, device=dev)
        fn = lambda: net.forward(imgs, lg, cls)  # noqa: E731
        ms, clocks = _timed_clocks(fn, a.steps, a.warmup)
        st, cnt = _stage_profile(net, fn)
        _, macs = conv_popc_per_image(synth.VEHICLE, mode)
        _emit({"metric": "images/s", "value": B / (ms * 1e-3), "unit": "images/s", "config": {
            "workload": "config 2: vehicle classifier, batch 4096, input binarization %s" % name},
            "ms_per_step": ms, "binary_or_int_mac_per_s": sum(macs) * B / (ms * 1e-3),
            "stage_ms": {("pack" if i == 0 else "layer%d" % (i - 1) if i <= 5 else "argmax"): round(x, 4)
                         for i, (x, c) in enumerate(zip(st, cnt)) if c},
            "layers": _layer_rooflines(net, synth.VEHICLE, mode, st, cnt, B, clocks), "clocks": clocks})
        net.close()


def run_alg1(a):
    """Speed-up context: the paper's own design (Alg. 1 im2col + packing, tiled XOR-popcount
    GEMM-conv, int32 max-pool, 64-segment FC; bnn_set_option("alg1", 1)) against this framework's path,
    same B200, same vehicle net (THRESH_RGB, no BN thresholds), batch 4096 and batch 1."""
    import torch
    import paper_1808_00209_b200 as bnn
    from paper_1808_00209_b200 import synth
    dev = torch.device("cuda", 0)
    B = 4096
    net, _, _ = _net_for(synth.VEHICLE, 1, a.seed, dev, B)
    imgs = synth.images(B, 96, 96, 3, a.seed + 1, device=dev)
    lg = torch.empty((B, 4), dtype=torch.int32, device=dev)
    cls = torch.empty((B,), dtype=torch.int32, device=dev)
    res = {}
    for name, flag in [("paper_alg1", 1), ("framework", 0)]:
        bnn.set_option("alg1", flag)
        fn = lambda: net.forward(imgs, lg, cls)  # noqa: E731
        ms, clocks = _timed_clocks(fn, a.steps, a.warmup)
        st, cnt = _stage_profile(net, fn)
        one = imgs[:1]
        lat = _timed(lambda: net.forward(one, lg[:1], cls[:1]), 200, 20) * 1e3
        res[name] = {"images_per_s": B / (ms * 1e-3), "ms_per_4096": ms, "batch1_us_stream": lat,
                     "stage_ms": [round(x, 4) for x, c in zip(st, cnt) if c], "clocks": clocks}
    bnn.set_option("alg1", 0)
    net.close()
    _emit({"metric": "images/s", "value": res["paper_alg1"]["images_per_s"], "unit": "images/s",
           "config": {"workload": "paper design (Alg. 1 + GEMM-conv + int32 max-pool + 64-segment FC) on the vehicle "
                                  "net, THRESH_RGB, batch 4096, same B200"},
           "paper_design": res["paper_alg1"], "framework": res["framework"],
           "speedup_framework_over_paper_design": res["framework"]["images_per_s"] / res["paper_alg1"]["images_per_s"],
           "clocks": res["framework"]["clocks"],
           "context": "paper Table 2 (GTX 1080, batch 1): 42.58 us binarized layers total (PAPER.md:325-331)"})


CIFAR_CHUNK = 8192  # images per internal chunk for config 4 (two chunks per 16384-image step)


def run_cifar(a):
    """BASELINE config 4: CIFAR-10-shaped BinaryNet VGG (reading R22), batch 16384, THRESH_RGB."""
    import torch
    from paper_1808_00209_b200 import synth
    dev = torch.device("cuda", 0)
    B = 16384
    net, _, _ = _net_for(synth.CIFAR, 1, a.seed, dev, CIFAR_CHUNK)
    imgs = synth.images(B, 32, 32, 3, a.seed + 1, device=dev)
    lg = torch.empty((B, 10), dtype=torch.int32, device=dev)
    cls = torch.empty((B,), dtype=torch.int32, device=dev)
    fn = lambda: net.forward(imgs, lg, cls)  # noqa: E731
    # the step is timed without per-kernel events (they serialise programmatic launches); per-layer
    # times come from a separate one-stream pass with the library's events
    ms, clocks = _timed_clocks(fn, a.steps, a.warmup)
    st, cnt = _stage_profile(net, fn)
    _, macs = conv_popc_per_image(synth.CIFAR, 1)
    _emit({"metric": "images/s", "value": B / (ms * 1e-3), "unit": "images/s", "config": {
        "workload": "config 4: CIFAR-10 BinaryNet VGG (2x128C3-MP2-2x256C3-MP2-2x512C3-MP2-1024FC-1024FC-10FC), "
                    "batch 16384, THRESH_RGB", "chunk": CIFAR_CHUNK}, "ms_per_step": ms,
        "binary_mac_per_s": sum(macs) * B / (ms * 1e-3),
        "layers": _layer_rooflines(net, synth.CIFAR, 1, st, cnt, B, clocks), "clocks": clocks})
    net.close()


def run_sweep(a):
    """BASELINE config 3: single binary conv layers, k in {3,5} x C in {64..1024} x H=W in {32..96},
    batch 256, C_out = C_in, sign threshold, no pool; inputs uniform random words.  Each point: the
    tensor roofline of its kernel (all run on tcgen05 kind::mxf4), the clocks over its timed region, and
    the packed output bits of 2 sampled pixels (every channel) against orc_conv_binary_point (Eq. 3 + Eq. 1)."""
    import numpy as np
    import torch
    import paper_1808_00209_b200 as bnn
    from oracle import oracle as orc
    from paper_1808_00209_b200 import synth
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    N = 256
    rng = np.random.default_rng(a.seed)
    for k in (3, 5):
        for C in (64, 128, 256, 512, 1024):
            ws = synth.pm1((C, k, k, C), a.seed + k + C)
            wt = bnn.pack_weights(ws.to(dev))
            ws_np = ws.numpy()
            for H in (32, 48, 64, 96):
                x = synth.words((N, H, H, C // 32), a.seed + H + C, device=dev)
                y = torch.empty((N, H, H, C // 32), dtype=torch.int32, device=dev)
                fn = lambda: bnn.conv2d(x, bnn.BITS, C, wt, C, k)  # noqa: E731
                ms, clocks = _timed_clocks(fn, 3, 1, 0.25)
                y, _ = fn()
                torch.cuda.synchronize()
                kernel = "conv_tc4_kernel" if (k == 5 and C <= 64) or (k == 3 and C in (64, 128)) else "conv_tc4_big_kernel"
                macs = N * H * H * C * k * k * C
                r = roofline_for(kernel, macs, macs / 32, ms, clocks, sms)
                # sampled parity: the last pixel of the last image and one random pixel, all C channels
                checks, ok = 0, True
                for (i, yy, xx) in [(N - 1, H - 1, H - 1), (int(rng.integers(N)), int(rng.integers(H)), int(rng.integers(H)))]:
                    # the k x k window (cropped at the map edge, so the -1 padding is the oracle's own)
                    R = k // 2
                    y0, x0 = max(0, yy - R), max(0, xx - R)
                    win = x[i, y0:min(H, yy + R + 1), x0:min(H, xx + R + 1)].cpu().numpy().view(np.uint32)
                    xi = orc.unpack_channels(win, C)
                    bits = np.array([orc.sign(orc.conv_binary_point(xi, ws_np[o], yy - y0, xx - x0))
                                     for o in range(C)], np.int8)
                    ok = ok and np.array_equal(y[i, yy, xx].cpu().numpy().view(np.uint32), orc.pack(bits))
                    checks += C
                _emit({"metric": "binary conv MAC/s", "value": macs / (ms * 1e-3), "unit": "binary MAC/s",
                       "config": {"workload": "config 3 sweep point", "k": k, "c": C, "hw": H, "batch": N,
                                  "kernel": kernel}, "ms": ms,
                       "roofline": {kk: r[kk] for kk in ("bound", "pipe", "unit", "achieved", "peak", "frac",
                                                         "peak_probe", "frac_probe", "peak_basis")},
                       "popc_equivalent_frac": r.get("popc_equivalent_frac"),
                       "parity": {"outputs_checked": checks, "bit_exact": bool(ok)}, "clocks": clocks})
                assert ok, "sweep point k=%d C=%d H=%d differs from the oracle" % (k, C, H)
                del x, y


if __name__ == "__main__":
    main()
