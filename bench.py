#!/usr/bin/env python3
"""Crossbar-evaluation hot path benchmark (BASELINE.json metric).

One step = one pass of the hot path over one batch: CrossbarCore forward
(K0a prep + K1 tcgen05 VMM), backward (K0b prep + K3a dW + K2 tcgen05 VMM)
and apply_updates (K3b fused update + regeneration) of the configs[1] layer
at its largest sweep point (M=256, K=N=4096, 128x128 crossbars, 8-bit in /
weights as four 2-bit slices, 1-bit DAC, 7-bit ADC, AAM parasitics).

  value : non-ideal crossbar MACs/s with inputs resident in HBM (device
          pointers through the C ABI), CUDA events on the core's stream,
          max over ranks; N ranks run N independent replicas (weak scaling).
  e2e   : the same metric through the host-pointer C-ABI calls (pinned host
          buffers; H2D of x, dy and D2H of y, dx inside every step).

`python bench.py --impl reference` times the reference algorithm's CPU
implementation (the restated oracle, oracle/ -- the reference itself cannot
be built here) on the host cores, on a bounded tile sample.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "non-ideal crossbar MACs/s (fwd+bwd+update) on 1 B200; % of int8 TC / HBM roofline"
L_LIMBS = 3  # u8 limbs per snapped conductance (three radix-255 digits, 24-bit grid) -> int8 ops = 2 * L * MAC


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c5", help="headline workload (default C5, the largest single-GPU config)")
    p.add_argument("--no-others", action="store_true", help="skip the per-config summaries of C1-C4")
    p.add_argument("--stage-probe", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-peak", action="store_true", help="skip the live int8 peak GEMM (ncu launch lists)")
    p.add_argument("--layer", type=int, default=0, help="layer index of a multi-layer config (default 0)")
    p.add_argument("--engine", default=None, choices=["aam", "fcm", "interp_fcm", "ideal"],
                   help="override the config's conversion engine")
    p.add_argument("--all-layers", action="store_true",
                   help="every layer of the config (C1/C3/C4 networks), one core per layer on one stream")
    p.add_argument("--traffic", default=None, help="json with ncu dram bytes per launch for the dominant kernel")
    p.add_argument("--calibrate", type=int, default=0, metavar="BATCHES",
                   help="ADC auto-calibration (SURVEY 8f row 3): adc.i_fs unset, BATCHES calibration steps, then "
                        "the freeze step and --steps quantised steps, each timed")
    p.add_argument("--conv", action="store_true",
                   help="C3/C4 as convolutions: CrossbarConv2d with device im2col/col2im (SURVEY 8f row 2)")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def init_dist(world, local_rank, backend):
    """One process per GPU (nccl) -- or per CPU rank (gloo, the CPU tests)."""
    if world <= 1:
        return
    import torch
    import torch.distributed as dist

    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        dist.init_process_group("gloo")


def max_over_ranks(x, world, device="cpu"):
    """Max of a per-rank scalar (device-timed ms) over all ranks."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.limit")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def start(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, pw, mx, plim, reasons = [], [], None, None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            try:
                pw.append(float(parts[2]))
            except ValueError:
                pw.append(float("nan"))
            try:
                plim = float(parts[8])
            except (ValueError, IndexError):
                pass
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        # "under load" = samples drawing at least half the window's peak power
        # (an idle SM sits at its max clock, so the clock alone cannot tell)
        pmax = max((p for p in pw if p == p), default=0.0)
        idx = [i for i, p in enumerate(pw) if pmax > 0 and p == p and p >= 0.5 * pmax] or list(range(len(sm)))
        loaded = [sm[i] for i in idx]
        out = {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
               "reasons": sorted(reasons), "samples": len(sm), "loaded_samples": len(loaded)}
        if pmax > 0:
            out["power_w"] = statistics.median([pw[i] for i in idx])
        if plim:
            out["power_limit_w"] = plim
        return out


# ------------------------------------------------------------ int8 peak
def measure_int8_peak():
    """Dense int8 tensor-core peak on this B200: torch._int_mm 8192^3 best of 10."""
    import torch

    try:
        n = 8192
        a = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-8, 8, (n, n), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(a, b)
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12, "measured: torch._int_mm 8192^3 best of 10 (TOPS)"
    except Exception as e:  # pragma: no cover
        return 4500.0, f"NVIDIA dense int8 spec 4.5 POPS (measurement failed: {e})"


# ----------------------------------------------------------- CPU baseline
def cpu_kind():
    """"reference": the reference's own core sources compiled in place
    against the Eigen-API shim (oracle/_ref, built where /root/reference
    exists and shipped with the snapshot); "port": the restated oracle."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_py

    return "reference" if ref_py.available() else "port"


def cpu_core(W, opt):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    if cpu_kind() == "reference":
        import ref_py

        T = opt.map.tile_rows
        return ref_py.RefCore(W, opt, T, opt.map.tile_cols, opt.map.num_slices(), 0)
    import oracle_py

    return oracle_py.OracleCore(W, opt, snapped=True)


CPU_NOTE = {"reference": ("the reference's core sources compiled unchanged against oracle/eigen_shim (no Eigen in the "
                          "image): its GEMMs run as ascending-order scalar loops, not Eigen's blocked kernels"),
            "port": "reference unbuildable here; restated oracle (snapped mode)"}


def cpu_sample(cfg, n_feat=256, steps=1, idx=0, rows=None):
    """The oracle (restated reference CPU path, 1 thread: the reference's
    forward/backward/update are serial, layers.hpp:34) on a bounded sample of
    the same workload: a K=N=n_feat slice of the layer (same tile geometry,
    batch, bits and options).  Returns (MAC/s, seconds, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from paper_2002_11151_b200.configs import Layer

    layer = cfg.layers[0]
    n_feat = min(n_feat, layer.K, layer.N)
    M = min(layer.M, rows or layer.M)
    sl = Layer("sample", M, n_feat, n_feat)
    opt = cfg.options()
    W, x, dy = cfg.weights(sl, idx), cfg.inputs(sl, idx), cfg.errors(sl, idx)
    orc = cpu_core(W, opt)
    t0 = time.perf_counter()
    for it in range(steps):
        orc.forward(x, True)
        orc.backward(dy, 1.0)
        orc.apply_updates(it)
    dt = (time.perf_counter() - t0) / steps
    macs = cfg.macs(sl)["total"]
    desc = (f"{cpu_kind()} fwd+bwd+update of a K=N={n_feat} slice of {cfg.name} ({M} of {layer.M} batch rows, "
            f"{(n_feat // cfg.tile) ** 2} of {((layer.K + cfg.tile - 1) // cfg.tile) * ((layer.N + cfg.tile - 1) // cfg.tile)}"
            f" crossbar tiles), {dt:.2f} s/step, MACs/s scale linearly in tile count")
    return macs / dt, dt, desc


def _ref_worker(a):
    from paper_2002_11151_b200.configs import CONFIGS

    name, idx = a
    cfg = CONFIGS[name]
    # bounded step: one crossbar tile's worth of the layer, at most 128 batch rows
    v, dt, desc = cpu_sample(cfg, cfg.tile, 1, idx, rows=128)
    return v * dt, desc  # MACs done, description


def run_reference(args, cfg):
    """The reference algorithm's CPU implementation on all host cores.  The
    reference's VMM loop is serial per core (threads only split regeneration,
    layers.hpp:34), so the whole-host rate is one independent one-tile slice
    of the workload (K = N = tile, <= 128 batch rows) per core, run
    concurrently: value = sum of MACs / wall time of the step.  Under
    torchrun only rank 0 runs."""
    import multiprocessing as mp

    rank, _, world = dist_env()
    if rank != 0:
        return
    ncores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    ctx = mp.get_context("fork")
    vals, desc = [], ""
    with ctx.Pool(ncores) as pool:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = pool.map(_ref_worker, [(args.config, 100 * i + w) for w in range(ncores)])
            dt = time.perf_counter() - t0
            desc = res[0][1]
            if i >= args.warmup:
                vals.append((sum(r[0] for r in res) / dt, dt))
    v = statistics.median([x[0] for x in vals]) if vals else 0.0
    dt = statistics.median([x[1] for x in vals]) if vals else 0.0
    sample = f"{ncores} concurrent processes, each: " + desc
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "MAC/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "layer": vars(cfg.layers[0]), "parallelism": f"cpu{ncores}"},
        "cpu_baseline": {"value": v, "unit": "MAC/s", "cores": ncores, "kind": cpu_kind(), "sample": sample,
                         "note": CPU_NOTE[cpu_kind()]},
        "e2e": {"value": v, "unit": "MAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- ours
def run_conv(args, cfg):
    """C3/C4 stepped as the reference's layer types: every conv layer a
    CrossbarConv2d (device im2col -> core -> col2im, layers.cpp:415-505),
    the fc a CrossbarLinear core, all on one stream with device tensors.
    Reports the same metric over the same MACs as --all-layers; the time the
    cores do not account for is the lowering glue."""
    import torch
    from paper_2002_11151_b200 import xbarsim as xb

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    init_dist(world, local_rank, "nccl")
    opt = cfg.options()
    mods, bufs = [], []
    for li, L in enumerate(cfg.layers):
        W = cfg.weights(L, li)
        cv = L.conv
        if cv is not None:
            m = xb.CrossbarConv2d(W, cv.in_c, cv.out_c, cv.k, cv.stride, cv.pad, opt)
            oh, ow = m.output_dims(cv.h, cv.w)
            n_in, n_out, batch = cv.in_c * cv.h * cv.w, cv.out_c * oh * ow, cv.batch
        else:
            m = xb.CrossbarCore(W, opt)
            n_in, n_out, batch = L.K, L.N, L.M
        g = torch.Generator().manual_seed(1000 + li)
        x = torch.randn((n_in, batch), generator=g, dtype=torch.float64).cuda()  # batch x n_in column-major
        dy = torch.randn((n_out, batch), generator=g, dtype=torch.float64).cuda()
        y = torch.empty((n_out, batch), dtype=torch.float64, device="cuda")
        dx = torch.empty((n_in, batch), dtype=torch.float64, device="cuda")
        mods.append(m)
        bufs.append((L, batch, x, dy, y, dx))
    cores = [m.core() if isinstance(m, xb.CrossbarConv2d) else m for m in mods]
    for c in cores[1:]:
        c.set_stream(cores[0].stream())
    stream = torch.cuda.ExternalStream(cores[0].stream())
    it = [0]

    def step():
        for m, (L, batch, x, dy, y, dx) in zip(mods, bufs):
            if L.conv is not None:
                m.forward_device(x.data_ptr(), batch, L.conv.in_c, L.conv.h, L.conv.w, True, y.data_ptr())
            else:
                m.forward_device(x.data_ptr(), batch, True, y.data_ptr())
        for m, (L, batch, x, dy, y, dx) in reversed(list(zip(mods, bufs))):
            if L.conv is not None:
                m.backward_device(dy.data_ptr(), batch, dx.data_ptr())
            else:
                m.backward_device(dy.data_ptr(), batch, 1.0, dx.data_ptr())
        for c in cores:
            c.apply_updates_device(it[0])
        it[0] += 1

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(world)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    for c in cores:
        c.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    e1.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, "cuda")
    core_ms = 0.0
    stages = {}
    for c in cores:
        for k, (t, n) in c.stage_times().items():
            stages[k] = stages.get(k, 0.0) + t / args.steps
            core_ms += t / args.steps
    clk = clocks.stop()
    for c in cores:
        c.profile(False)
    macs = 0
    for L in cfg.layers:
        macs += cfg.macs(L)["total"]
    e2e = None
    if not args.no_e2e:
        # the same step through the host-pointer C ABI (xbs_conv2d_forward /
        # _backward, xbs_core_forward / _backward for the fc): every layer's
        # images / errors copied in from pinned host memory and its outputs /
        # input gradients copied out, inside the timed region
        def pinned(rows, cols):  # F-ordered (rows x cols) numpy view of pinned memory
            return torch.empty((cols, rows), dtype=torch.float64, pin_memory=True).numpy().T

        hb, bi, bo = [], 0, 0
        for m, (L, batch, x, dy, y, dx) in zip(mods, bufs):
            hx, hdy = pinned(batch, x.shape[0]), pinned(batch, dy.shape[0])
            hy, hdx = pinned(batch, y.shape[0]), pinned(batch, dx.shape[0])
            hx[:] = x.cpu().numpy().T
            hdy[:] = dy.cpu().numpy().T
            hb.append((hx, hdy, hy, hdx))
            bi += 8 * batch * (x.shape[0] + dy.shape[0])
            bo += 8 * batch * (y.shape[0] + dx.shape[0])

        def host_step():
            for m, (L, batch, x, dy, y, dx), (hx, hdy, hy, hdx) in zip(mods, bufs, hb):
                if L.conv is not None:
                    m.forward(xb.Tensor(hx, [L.conv.in_c, L.conv.h, L.conv.w]), True, out=hy)
                else:
                    m.forward(hx, True, out=hy)
            for m, (L, batch, x, dy, y, dx), (hx, hdy, hy, hdx) in reversed(list(zip(mods, bufs, hb))):
                if L.conv is not None:
                    m.backward(xb.Tensor(hdy, [hdy.shape[1]]), out=hdx)
                else:
                    m.backward(hdy, 1.0, out=hdx)
            for m in mods:
                m.apply_updates(it[0])
            it[0] += 1

        for _ in range(max(3, args.warmup)):
            host_step()
        for c in cores:
            c.synchronize()
        barrier(world)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        f0.record(stream)
        for _ in range(args.steps):
            host_step()
        f1.record(stream)
        f1.synchronize()
        wall = (time.perf_counter() - t0) / args.steps
        e_ms = max_over_ranks(f0.elapsed_time(f1) / args.steps, world, "cuda")
        e2e = {"value": world * macs / (e_ms * 1e-3), "unit": "MAC/s", "h2d_bytes_per_step": bi,
               "d2h_bytes_per_step": bo, "ms_per_step": e_ms, "wall_ms_per_step": max_over_ranks(wall * 1e3, world, "cuda"),
               "path": "xbs_conv2d_forward/backward + xbs_core_forward/backward (fc), apply_updates "
                       "(host pointers, pinned): images, not patch matrices, cross PCIe"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": world * macs / (ms * 1e-3), "unit": "MAC/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic N(0,1) images and errors",
            "config": {"workload": cfg.name.replace("-im2col", "") + "-conv",
                       "lowering": "CrossbarConv2d: device im2col / col2im around one core per layer",
                       "layers": [[L.name, L.M, L.K, L.N] for L in cfg.layers], "parallelism": f"replicas{world}"},
            "stage_ms": stages, "core_ms": core_ms, "glue_ms": ms - core_ms, "clocks": clk}
        if e2e:
            line["e2e"] = e2e
        print(json.dumps(line))
    for c in cores[1:]:  # the first core owns the shared stream: detach before teardown
        c.set_stream(None)
    torch.cuda.synchronize()
    del cores
    while mods:
        mods.pop()


def run_calibrate(args, cfg):
    """ADC auto-calibration on the device: pass-through calibration steps
    (currents recorded), the freeze (exact nearest-rank select over the
    record), then quantised steps.  Every layer of the config, one stream."""
    import torch
    from paper_2002_11151_b200 import xbarsim as xb

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    init_dist(world, local_rank, "nccl")
    opt = cfg.options()
    opt.adc.i_fs = 0.0
    opt.adc_cal_batches = args.calibrate
    cores, dev = [], []
    for li, L in enumerate(cfg.layers):
        cores.append(xb.CrossbarCore(cfg.weights(L, li), opt))
        x, dy = cfg.inputs(L, li), cfg.errors(L, li)
        dev.append((L, torch.from_numpy(np.ascontiguousarray(x.T)).cuda(),
                    torch.from_numpy(np.ascontiguousarray(dy.T)).cuda(),
                    torch.empty((L.N, L.M), dtype=torch.float64, device="cuda"),
                    torch.empty((L.K, L.M), dtype=torch.float64, device="cuda")))
    for c in cores[1:]:
        c.set_stream(cores[0].stream())
    it = [0]

    def step():
        for c, (L, x, dy, y, dx) in zip(cores, dev):
            c.forward_device(x.data_ptr(), L.M, True, y.data_ptr())
        for c, (L, x, dy, y, dx) in reversed(list(zip(cores, dev))):
            c.backward_device(dy.data_ptr(), L.M, 1.0, dx.data_ptr())
        for c in cores:
            c.apply_updates_device(it[0])
        it[0] += 1

    def timed(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            step()
        for c in cores:
            c.synchronize()
        return (time.perf_counter() - t0) * 1e3 / max(1, n)

    cal_ms = timed(args.calibrate)       # pass-through, currents recorded
    freeze_ms = timed(1)                 # freeze (select) + first quantised step
    q_ms = timed(args.steps)
    macs = sum(cfg.macs(L)["total"] for L in cfg.layers)
    fs = [c.forward_adc_full_scale() for c in cores]
    for c in cores[1:]:
        c.set_stream(None)
    if rank == 0:
        print(json.dumps({
            "metric": "ADC auto-calibration step time", "unit": "ms", "higher_is_better": False,
            "n_gpus": world, "steps": args.steps, "warmup": 0, "data": "synthetic",
            "config": {"workload": cfg.name + "-autocal", "adc_cal_batches": args.calibrate,
                       "layers": [[L.M, L.K, L.N] for L in cfg.layers]},
            "calibration_step_ms": cal_ms, "freeze_step_ms": freeze_ms, "quantised_step_ms": q_ms,
            "quantised_macs_per_s": macs / (q_ms * 1e-3), "frozen_forward_i_fs": fs,
            "timing": "host wall clock around synchronised steps"}))


MMA_SPEC_TOPS = 4500.0  # NVIDIA dense int8 spec (B200)
OTHER_CONFIGS = ("c1", "c2-4096", "c3", "c4")


def stage_work(cfg, layers, S):
    """Algorithmic work per step of each stage."""
    macs = {}
    for L in layers:
        for k, v in cfg.macs(L).items():
            macs[k] = macs.get(k, 0) + v
    return macs, {
        "fwd_vmm": ("tensor", 2 * L_LIMBS * macs["fwd"] / 1e12, "TFLOP/s"),
        "bwd_vmm": ("tensor", 2 * L_LIMBS * macs["bwd"] / 1e12, "TFLOP/s"),
        # dW: an M-deep outer product whose cost is writing K x N fp64 and
        # reading the u8 codes -- HBM-bound
        "dw": ("hbm", sum(8 * L.K * L.N + L.M * (L.K + 2 * L.N) for L in layers) / 1e9, "GB/s"),
        # fp64 master read + write, both polarities' VMM-ready digits (L bytes
        # each), dW read once (24 S + 8 at L = 4)
        "update": ("hbm", sum(L.K * L.N * ((16 + 2 * L_LIMBS) * S + 8) for L in layers) / 1e9, "GB/s"),
        # input / error quantisation + bit-plane emission: read fp64, write
        # codes and the two u8 plane copies (x: T_in planes; dy: 2 T_err)
        "prep_x": ("hbm", sum(L.M * L.K * (8 + 2 + 1 + 2 * 8) for L in layers) / 1e9, "GB/s"),
        "prep_dy": ("hbm", sum(L.M * L.N * (8 + 2 + 2 + 4 * 8) for L in layers) / 1e9, "GB/s"),
    }


def measure(args, cfg, layers, world, local_rank, steps, warmup, e2e=True, profile=True, engine=None):
    """One core per layer on one stream; W warm-up steps, K device-resident
    steps timed with CUDA events on the cores' stream (graph replays), then
    K profiled steps for per-stage times, then (e2e) K steps through the
    host-pointer C ABI with pinned buffers.  Returns a dict of raw numbers."""
    import torch
    from paper_2002_11151_b200 import xbarsim as xb

    opt = cfg.options()
    if engine:
        opt.engine = getattr(xb.EngineKind, engine)
    cores, host, dev = [], [], []
    for li, layer in enumerate(layers):
        W, x, dy = cfg.weights(layer, li), cfg.inputs(layer, li), cfg.errors(layer, li)
        cores.append(xb.CrossbarCore(W, opt))
        host.append((x, dy) if e2e else None)
        # device-resident operands, column-major (Eigen layout): (K, M) C-order == M x K col-major
        dev.append((torch.from_numpy(np.ascontiguousarray(x.T)).cuda(),
                    torch.from_numpy(np.ascontiguousarray(dy.T)).cuda(),
                    torch.empty((layer.N, layer.M), dtype=torch.float64, device="cuda"),
                    torch.empty((layer.K, layer.M), dtype=torch.float64, device="cuda")))
        del W, x, dy
    for c in cores[1:]:
        c.set_stream(cores[0].stream())  # one stream for the whole network
    stream = torch.cuda.ExternalStream(cores[0].stream())
    torch.cuda.synchronize()
    it = [0]

    def step():
        for c, layer, (d_x, d_dy, d_y, d_dx) in zip(cores, layers, dev):
            c.forward_device(d_x.data_ptr(), layer.M, True, d_y.data_ptr())
        for c, layer, (d_x, d_dy, d_y, d_dx) in reversed(list(zip(cores, layers, dev))):
            c.backward_device(d_dy.data_ptr(), layer.M, 1.0, d_dx.data_ptr())
        for c in cores:
            c.apply_updates_device(it[0])
        it[0] += 1

    for _ in range(warmup):
        step()
    for c in cores:
        c.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    out = {}
    launches0 = sum(c.launch_count() for c in cores)
    fb0 = sum(int(c.info().tc_fallbacks) for c in cores)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    e1.synchronize()
    for c in cores:
        c.synchronize()
    torch.cuda.synchronize()
    out["ms"] = max_over_ranks(e0.elapsed_time(e1) / steps, world, "cuda")
    out["launches"] = sum(c.launch_count() for c in cores) - launches0
    out["fallbacks"] = sum(int(c.info().tc_fallbacks) for c in cores) - fb0
    # per-stage kernel times: the same K steps again with CUDA events around
    # every stage (eager launches; the timed steps above replay the cores'
    # captured graphs, which per-stage events would split)
    stages = {}
    if profile:
        for c in cores:
            c.profile(True)
        for _ in range(steps):
            step()
        for c in cores:
            c.synchronize()
        for c in cores:
            for k, (t, n) in c.stage_times().items():
                t0, n0 = stages.get(k, (0.0, 0))
                stages[k] = (t0 + t, n0 + n)
            c.profile(False)
    out["stages_ms"] = {k: (v[0] / v[1] * len(layers) if v[1] else 0.0) for k, v in stages.items()}
    barrier(world)
    if e2e:
        def pinned(rows, cols):  # F-ordered (rows x cols) numpy view of pinned memory
            return torch.empty((cols, rows), dtype=torch.float64, pin_memory=True).numpy().T

        hbuf = []
        for layer, (x, dy) in zip(layers, host):
            hx, hdy, hy, hdx = pinned(layer.M, layer.K), pinned(layer.M, layer.N), pinned(layer.M, layer.N), pinned(
                layer.M, layer.K)
            hx[:] = x
            hdy[:] = dy
            hbuf.append((hx, hdy, hy, hdx))
        host.clear()

        def host_step():
            for c, (hx, hdy, hy, hdx) in zip(cores, hbuf):
                c.forward(hx, True, out=hy)
            for c, (hx, hdy, hy, hdx) in reversed(list(zip(cores, hbuf))):
                c.backward(hdy, 1.0, out=hdx)
            for c in cores:
                c.apply_updates(it[0])
            it[0] += 1

        for _ in range(max(3, warmup)):
            host_step()
        for c in cores:
            c.synchronize()
        barrier(world)
        # the host calls are synchronous; events on the (shared) stream
        # bracket every H2D copy, kernel and D2H copy of the K steps
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        f0.record(stream)
        for _ in range(steps):
            host_step()
        f1.record(stream)
        f1.synchronize()
        wall_s = (time.perf_counter() - t0) / steps
        bi = sum(8 * L.M * (L.K + L.N) for L in layers)
        out["e2e"] = {"h2d_bytes_per_step": bi, "d2h_bytes_per_step": bi,
                      "s": max_over_ranks(f0.elapsed_time(f1) * 1e-3 / steps, world, "cuda"),
                      "wall_s": max_over_ranks(wall_s, world, "cuda")}
        out["fallbacks"] += sum(int(c.info().tc_fallbacks) for c in cores) - fb0 - out["fallbacks"]
    for c in cores[1:]:  # the first core owns the shared stream: detach before teardown
        c.set_stream(None)
    torch.cuda.synchronize()
    del cores, dev
    torch.cuda.empty_cache()
    return out


def rooflines(cfg, layers, stages_ms, peak_tops, hbm, mma_only=None):
    S = cfg.weight_bits // cfg.device_bits
    macs, work = stage_work(cfg, layers, S)
    conv = {}
    for L in layers:
        for k, v in cfg.adc_conversions(L).items():
            conv[k] = conv.get(k, 0) + v
    roof = {}
    for st, (bound, amount, unit) in work.items():
        ms = stages_ms.get(st)
        if not ms:
            continue
        ach = amount / (ms * 1e-3)
        pk = peak_tops if bound == "tensor" else hbm
        roof[st] = {"bound": bound, "achieved": ach, "peak": pk, "unit": unit, "frac": ach / pk, "ms": ms}
        if st in ("fwd_vmm", "bwd_vmm"):
            # the ADC epilogue's work: conversions/s and MACs per conversion
            # (the tensor fraction of a narrow layer is capped by the latter)
            n = conv[st[:3]]
            roof[st].update({"adc_conversions": n, "adc_conv_per_s": n / (ms * 1e-3),
                             "macs_per_conversion": macs[st[:3]] / n,
                             "frac_vs_spec": ach / MMA_SPEC_TOPS})
            if mma_only and mma_only.get(st):
                mo = amount / (mma_only[st] * 1e-3)
                roof[st].update({"mma_only_rate": mo, "frac_vs_mma_only": ach / mo})
        if st == "update" and cfg.sigma != 0.0:
            # sigma != 0: the kernel also streams the cached fp64 variation
            # multipliers of both polarities (16 B per device and slice; the
            # reference re-derives them from the counter RNG each
            # regeneration, which costs more fp64 time on B200 than reading
            # them -- DESIGN.md section 4)
            moved = amount + sum(L.K * L.N * 16 * S for L in layers) / 1e9
            roof[st].update({"bytes_moved_gb": moved, "achieved_moved": moved / (ms * 1e-3),
                             "frac_moved": moved / (ms * 1e-3) / hbm})
    return macs, roof


def mma_only_probe(args, cfg_name):
    """Per-stage VMM times of this workload with the ADC epilogue stubbed out
    (the XBS_STUB_EPI build, _lib_stubepi/: MMAs, TMA operand loads, TMEM
    loads and barriers, no conversions) -- the rate this kernel design reaches
    without the epilogue.  Runs in a child process (the library is loaded per
    process); None when the stub build is absent."""
    lib = os.path.join(ROOT, "paper_2002_11151_b200", "_lib_stubepi", "libxbarsim_b200.so")
    if not os.path.exists(lib):
        return None
    env = dict(os.environ, XBS_LIB_PATH=lib)
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--config", cfg_name, "--stage-probe",
                        "--steps", "3", "--warmup", "2"], env=env, capture_output=True, text=True, timeout=900)
    try:
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        return None


def main():
    args = parse()
    from paper_2002_11151_b200.configs import CONFIGS

    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    if args.conv:
        run_conv(args, cfg)
        return
    if args.calibrate:
        run_calibrate(args, cfg)
        return

    import torch

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    if args.stage_probe:  # child of mma_only_probe: stage times only
        layers = list(cfg.layers)
        r = measure(args, cfg, layers, 1, local_rank, args.steps, args.warmup, e2e=False)
        print(json.dumps(r["stages_ms"]))
        return
    init_dist(world, local_rank, "nccl")

    layers = list(cfg.layers) if (args.all_layers or len(cfg.layers) == 1) else [cfg.layers[args.layer]]
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    r = measure(args, cfg, layers, world, local_rank, args.steps, args.warmup, e2e=not args.no_e2e,
                engine=args.engine)
    clk = clocks.stop()
    if r["fallbacks"]:  # a VMM left the tcgen05 kernels (exact SIMT ran): not a tensor-core measurement
        print(json.dumps({"error": f"{r['fallbacks']} tcgen05->SIMT VMM fallbacks during the bench",
                          "config": cfg.name}), file=sys.stderr)
        sys.exit(3)

    S = cfg.weight_bits // cfg.device_bits
    peak_tops, peak_src = (MMA_SPEC_TOPS, "NVIDIA dense int8 spec (--no-peak)") if args.no_peak else measure_int8_peak()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    mma_only = None if (args.no_peak or world > 1) else mma_only_probe(args, args.config)
    macs, roof_all = rooflines(cfg, layers, r["stages_ms"], peak_tops, hbm, mma_only)
    per = r["stages_ms"]
    dominant = max(("fwd_vmm", "bwd_vmm", "update", "dw", "prep_x", "prep_dy"), key=lambda s: per.get(s, 0.0))
    traffic = None
    tpath = args.traffic or os.path.join(ROOT, "profiles", f"traffic_{cfg.name}.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(dominant)
    roof = dict(roof_all.get(dominant, {}))
    roof.update({"kernel": dominant, "traffic": traffic,
                 "peak_source": peak_src if roof.get("bound") == "tensor" else "MEASURED_PEAKS.json hbm_gbs"})

    ms = r["ms"]
    value = world * macs["total"] / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "MAC/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": dict(
            {"workload": cfg.name, "tile": cfg.tile, "slices": S, "adc_bits": cfg.adc_bits,
             "parallelism": f"replicas{world}",
             "l2": "conductance digits %.0f MB read per pass (L2 126 MB)" % (
                 sum(2 * S * L.K * L.N * 4 for L in layers) / 1e6)},
            **({"layers": [[L.M, L.K, L.N] for L in layers]} if len(layers) > 1 else
               {"M": layers[0].M, "K": layers[0].K, "N": layers[0].N})),
        "roofline": roof,
        "roofline_stages": roof_all,
        "int8_peak_tops": peak_tops,
        "int8_peak_denominators": {"live_int_mm": peak_tops, "spec": MMA_SPEC_TOPS,
                                   "mma_only_stub_ms": mma_only},
        "macs_per_step": macs,
        "gpu_launches": r["launches"],
        "tc_fallbacks": r["fallbacks"],
        "clocks": clk,
    }
    if "e2e" in r:
        e = r["e2e"]
        line["e2e"] = {"value": world * macs["total"] / e["s"], "unit": "MAC/s",
                       "h2d_bytes_per_step": e["h2d_bytes_per_step"], "d2h_bytes_per_step": e["d2h_bytes_per_step"],
                       "ms_per_step": e["s"] * 1e3, "wall_ms_per_step": e["wall_s"] * 1e3,
                       "path": "xbs_core_forward/backward/apply_updates (host pointers, pinned)"}
    fl = os.path.join(ROOT, "profiles", "r02", "adc_flips.json")
    if os.path.exists(fl):
        f = json.load(open(fl))
        line["parity"] = {"gpu_vs_snapped_oracle": "bit-exact y, dx, dW (tests/test_parity*_gpu.py, "
                                                   "tests/test_adc_flips_gpu.py)",
                          "adc_flips_vs_literal": {"total": f["total"], "max_abs_code_delta": f["max_abs_code_delta"],
                                                   "source": "profiles/r02/adc_flips.json (tools/flip_report.py)"}}
    if not args.no_others:
        others = {}
        for name in OTHER_CONFIGS:
            if name == args.config:
                continue
            oc = CONFIGS[name]
            ol = list(oc.layers)
            o = measure(args, oc, ol, world, local_rank, min(args.steps, 10), max(3, min(args.warmup, 5)), e2e=False)
            om, orf = rooflines(oc, ol, o["stages_ms"], peak_tops, hbm)
            others[oc.name] = {"value": world * om["total"] / (o["ms"] * 1e-3), "unit": "MAC/s", "ms_per_step": o["ms"],
                               "layers": len(ol), "tc_fallbacks": o["fallbacks"],
                               "frac": {k: round(v["frac"], 4) for k, v in orf.items()},
                               "stage_ms": {k: round(v, 4) for k, v in o["stages_ms"].items()}}
        line["other_configs"] = others
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, desc = cpu_sample(cfg, 256, 2, rows=512)
        line["cpu_baseline"] = {"value": v, "unit": "MAC/s", "cores": 1, "kind": cpu_kind(),
                                "sample": desc + f"; 2 steps, {2 * dt:.1f} s of CPU work", "note": CPU_NOTE[cpu_kind()]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
