#!/usr/bin/env python
"""Benchmark: Jagged Flash Attention fwd+bwd, useful TFLOP/s (BASELINE.json configs[2] = "cfg3").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

`python bench.py --gpus N` with N > 1 outside torchrun re-launches itself through torch.distributed.run with N
ranks (one per GPU, NCCL), so both launch forms measure N GPUs.

A step = one jagged_flash_attention_forward + jagged_flash_attention_backward over the rank's
shard of the batch (B=1024 per GPU, max_len=1024, D=128, H=4, bf16, half-mean lengths seed 0).
Useful FLOPs = 14·H·D·ΣBi² per step (fwd 4·H·D·ΣBi², bwd 10·H·D·ΣBi²; padding never counted).
Weak scaling: the global batch is 1024·N samples, sharded on Bi²-balanced sample boundaries, no
collective inside the timed region. Inputs (537 MB per tensor) are larger than L2. With N > 1 a verification
leg follows the timing: rank 0 scatters a verification batch (offsets by broadcast, shard rows by
point-to-point sends over NCCL), every rank runs fwd+bwd on its shard, the outputs, lse and grads are gathered
back to rank 0 and compared bit for bit with rank 0's single-GPU recomputation of every shard, and within the
bf16 tolerance with its single-GPU run of the whole batch ("verify").

--impl reference times the reference's own CPU implementation (oracle/_ref, compiled from the
reference sources) on the host cores, on bounded samples of the same workload.
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

METRIC = "Jagged flash-attn fwd+bwd TFLOP/s (useful FLOPs), 1–8 B200; jagged-op GB/s"
CFG = dict(batch_per_gpu=1024, max_len=1024, head_dim=128, heads=4, dist="half-mean", seed=0)


def useful_flops(lengths, H, D):
    sq = int((np.asarray(lengths, np.int64) ** 2).sum())
    return 4 * H * D * sq, 10 * H * D * sq, sq


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), \
            float(d["hbm_gbs"]), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


# ------------------------------------------------------------------ clocks sampler
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sync_boost", 0x40: "sw_thermal_slowdown", 0x80: "hw_thermal_slowdown",
               0x100: "hw_power_brake_slowdown", 0x200: "display_clock_setting"}


class Clocks:
    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except (FileNotFoundError, OSError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.rows.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if not self.rows:
            return None
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for r in self.rows for bit, name in REASON_BITS.items() if r[2] & bit} - {"gpu_idle"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU reference timing
def _cpu_kind():
    from oracle import reference as F

    return ("reference", F.hardware_threads()) if F.available() else ("port", 1)


def _cpu_run(lengths, D, stride, kind, threads):
    """One fwd+bwd of the reference CPU JFA (oracle/_ref when built, else the C port) on every
    stride-th non-empty sample, one head, fp32 instantiation. Returns (seconds, flops, samples)."""
    from oracle import reference as F
    from oracle import restated as Rr

    ln = np.asarray(lengths, np.int64)[::stride]
    ln = ln[ln > 0]
    off = np.concatenate([[0], np.cumsum(ln)]).astype(np.int64)
    S = int(off[-1])
    rng = np.random.default_rng(0)
    q, k, v, go = (rng.uniform(-1, 1, (S, D)).astype(np.float32) for _ in range(4))
    t0 = time.perf_counter()
    if kind == "reference":
        o, lse = F.jfa_forward(off, q, k, v, 64, 64, prec="f32", threads=threads)
        F.jfa_backward(off, q, k, v, go, o, lse, 64, 64, prec="f32", threads=threads)
    else:
        o, lse = Rr.jfa_forward(off, q.astype(np.float64), k.astype(np.float64), v.astype(np.float64))
        Rr.jfa_backward(off, q, k, v, go, o, lse)
    return time.perf_counter() - t0, 14 * D * int((ln * ln).sum()), len(ln)


def calibrate_stride(lengths, D, target_s, kind, threads):
    stride = 256
    dt, fl, n = _cpu_run(lengths, D, stride, kind, threads)
    while dt < target_s / 3 and stride > 1:  # grow the sample to ~target_s of CPU work
        stride = max(1, int(stride * max(dt, 1e-3) / target_s))
        stride = 1 << int(np.floor(np.log2(stride)))
        dt, fl, n = _cpu_run(lengths, D, stride, kind, threads)
    return stride, dt, fl, n


def cpu_reference_sample(lengths, H, D, target_s: float):
    kind, threads = _cpu_kind()
    stride, dt, fl, n = calibrate_stride(lengths, D, target_s, kind, threads)
    return dict(value=fl / dt / 1e12, unit="TFLOP/s", cores=int(threads), kind=kind,
                sample=f"every {stride}th sample of cfg3 ({n} samples, 1 of {H} heads, D={D}), fp32 "
                       f"instantiation, fwd+bwd, {dt:.1f} s wall, KernelOptions.threads={threads}",
                seconds=dt, stride=stride)


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from paper_2409_15373_b200 import synth

    L, D, H = CFG["max_len"], CFG["head_dim"], CFG["heads"]
    lengths = synth.gen_lengths(CFG["dist"], L, CFG["seed"], CFG["batch_per_gpu"] * world)
    kind, threads = _cpu_kind()
    budget = min(10.0, 150.0 / max(1, args.steps + args.warmup))  # whole run within a few minutes
    stride, _, _, _ = calibrate_stride(lengths, D, budget, kind, threads)
    times = []
    for it in range(args.warmup + args.steps):
        dt, fl, n = _cpu_run(lengths, D, stride, kind, threads)
        if it >= args.warmup:
            times.append((fl / dt / 1e12, dt, n))
    v = float(np.median([t[0] for t in times]))
    secs = float(np.median([t[1] for t in times]))
    probe = {"cores": threads, "kind": kind,
             "sample": f"every {stride}th sample of cfg3 ({times[0][2]} samples, 1 of {H} heads, D={D}) per step, "
                       f"fp32 instantiation, fwd+bwd, KernelOptions.threads={threads}"}
    times = [probe]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "cfg3: JFA fwd+bwd B=1024/GPU L=1024 D=128 H=4 half-mean seed 0 (bounded sample)",
                       "global_batch": int(len(lengths))},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": probe["cores"], "kind": probe["kind"],
                             "sample": probe["sample"]},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def verify_sharded(world, rank, dev, n_samples=64):
    """SURVEY §8e verification over NCCL: scatter a cfg3-shaped verification batch from rank 0, compute each
    shard's fwd+bwd, gather outputs / lse / grads to rank 0 and compare with rank 0's unsharded run (every sample
    depends only on its own rows and the backward is deterministic, so the results must be bit-identical)."""
    import torch
    import torch.distributed as dist

    from paper_2409_15373_b200 import shard, synth
    from paper_2409_15373_b200 import jagged as J

    L, D, H = CFG["max_len"], CFG["head_dim"], CFG["heads"]
    ln = synth.gen_lengths(CFG["dist"], L, CFG["seed"] + 7, n_samples * world)
    off = synth.offsets_of(ln)
    S = int(off[-1])
    full = None
    if rank == 0:
        g = torch.Generator(device=dev).manual_seed(123)
        full = (torch.rand(4, S, H, D, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
    probe = torch.empty(0, H, D, dtype=torch.bfloat16, device=dev)
    # scatter the four operands (q, k, v, grad_out) as one [rows, 4, H, D] tensor: one transfer per rank
    stacked = full.permute(1, 0, 2, 3).contiguous() if rank == 0 else probe.new_empty(0, 4, H, D)
    sh, loc = shard.scatter_jagged(off, stacked, world, rank, cost="sq", src=0)
    T = lambda a, o: J.JaggedTensor(torch.from_numpy(o).to(dev), a.contiguous(), o)  # noqa: E731
    lo = sh.offsets
    Q, K, V, G = (T(loc[:, i], lo) for i in range(4))
    s = J.jagged_flash_attention_forward(Q, K, V)
    gr = J.jagged_flash_attention_backward(Q, K, V, G, s)
    outs = torch.stack([s.output.values, gr.dq.values, gr.dk.values, gr.dv.values], 1)  # [rows, 4, H, D]
    lse = s.logsumexp.t().contiguous()                                                  # [rows, H]
    g_out = shard.gather_jagged(sh, outs, off, world, rank, cost="sq", dst=0)
    g_lse = shard.gather_jagged(sh, lse, off, world, rank, cost="sq", dst=0)
    torch.cuda.synchronize()
    if rank != 0:
        return None
    def run(o, rows):  # fwd + bwd of the rows [rows] of `full` with (rebased) offsets o, outputs stacked
        Qf, Kf, Vf, Gf = (T(full[i, rows], o) for i in range(4))
        sf = J.jagged_flash_attention_forward(Qf, Kf, Vf)
        gf = J.jagged_flash_attention_backward(Qf, Kf, Vf, Gf, sf)
        return (torch.stack([sf.output.values, gf.dq.values, gf.dk.values, gf.dv.values], 1),
                sf.logsumexp.t().contiguous())

    # bit-exact check: rank 0 recomputes every shard on its own rebased offsets (same inputs, same kernels, same
    # schedule shape) and the gathered results must equal it bit for bit (the transport is exact and the backward
    # deterministic). The whole-batch run is compared within the bf16 tolerance: the short-sample forward packing
    # groups samples by their position in the flat row space, so moving a shard boundary may regroup them and
    # change the last bits of a packed row's sums.
    b = shard.shard_bounds(ln, world, "sq")
    parts = [run(off[b[r]:b[r + 1] + 1] - off[b[r]], slice(int(off[b[r]]), int(off[b[r + 1]]))) for r in range(world)]
    ref_out = torch.cat([x[0] for x in parts], 0)
    ref_lse = torch.cat([x[1] for x in parts], 0)
    same = bool(torch.equal(g_out, ref_out)) and bool(torch.equal(g_lse, ref_lse))
    whole_out, _ = run(off, slice(0, S))
    diff = float((g_out.float() - whole_out.float()).abs().max()) if S else 0.0
    return {"samples": int(len(ln)), "rows": S, "ranks": world, "collective": dist.get_backend(),
            "shards_rows": [int(x) for x in np.diff(off[b])],
            "bit_identical": same, "max_abs_vs_unsharded": diff, "unsharded_match": diff <= 2e-2}


def run_ours(args, rank, world, local_rank):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2409_15373_b200 import _lib, shard, synth
    from paper_2409_15373_b200 import jagged as J

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, D, H = CFG["max_len"], CFG["head_dim"], CFG["heads"]
    lengths_all = synth.gen_lengths(CFG["dist"], L, CFG["seed"], CFG["batch_per_gpu"] * world)
    sh = shard.make_shard(lengths_all, world, rank, cost="sq")
    ln = sh.lengths
    off = sh.offsets
    S = int(off[-1])
    fwd_fl, bwd_fl, sq = useful_flops(ln, H, D)
    tot_fwd, tot_bwd, tot_sq = useful_flops(lengths_all, H, D)

    g = torch.Generator(device=dev).manual_seed(1 + rank)
    mk = lambda: (torch.rand(S, H, D, device=dev, generator=g, dtype=torch.float32) * 2 - 1).to(torch.bfloat16)  # noqa
    q, k, v, go = mk(), mk(), mk(), mk()
    T = lambda a: J.JaggedTensor(torch.from_numpy(off).to(dev), a, off)  # noqa: E731
    Q, K, V, G = T(q), T(k), T(v), T(go)
    sched = J.Schedule(Q)
    lib = _lib.lib()
    ws = torch.empty(J.backward_workspace_size(Q), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step(evs=None):
        if evs:
            evs[0].record(stream)
        saved = J.jagged_flash_attention_forward(Q, K, V, 64, 64, schedule=sched)
        if evs:
            evs[1].record(stream)
        J.jagged_flash_attention_backward(Q, K, V, G, saved, schedule=sched, workspace=ws)
        if evs:
            evs[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local_rank)
    clocks.start()
    time.sleep(0.3)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    lib.jg_reset_launch_count()
    t0.record(stream)
    for s in range(args.steps):
        step(evs[s])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = int(lib.jg_launch_count())
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = t0.elapsed_time(t1)
    fwd_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    bwd_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
    step_ms = [e[0].elapsed_time(e[2]) for e in evs]  # per-step spread (median with p10/p90)

    # e2e through the host-buffer C-ABI entry point (pinned host memory, H2D + compute + D2H)
    hq, hk, hv, hg = (t.cpu().pin_memory() for t in (q, k, v, go))
    ho, hdq, hdk, hdv = (torch.empty_like(hq).pin_memory() for _ in range(4))
    hl = torch.empty(H, S, dtype=torch.float32).pin_memory()
    hoff = np.ascontiguousarray(off, np.int64)
    e2e_steps = max(1, min(args.steps, 5))

    def e2e_call():
        _lib.check(lib.jg_jagged_flash_attention_fwd_bwd_host(
            hoff.ctypes.data, len(hoff) - 1, H, D, hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), hg.data_ptr(),
            ho.data_ptr(), hl.data_ptr(), hdq.data_ptr(), hdk.data_ptr(), hdv.data_ptr(), 1, stream.cuda_stream))

    e2e_s = float("nan")
    if not args.no_e2e:
        e2e_call()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t_e2e = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_call()
        e2e_s = (time.perf_counter() - t_e2e) / e2e_steps
    h2d = 4 * hq.numel() * 2 + hoff.nbytes
    d2h = 4 * hq.numel() * 2 + hl.numel() * 4

    verify = verify_sharded(world, rank, dev) if world > 1 else None  # after the timed regions

    # fp32 mode (the reference's float instantiation, attention.cpp:311-331) on the same shard, after the timed
    # regions: the split-bf16 tcgen05 kernels (attn_x3_sm100.cu); reported beside the bf16 headline, not in it
    fp32 = None
    if not args.no_fp32 and rank == 0:
        Qf, Kf, Vf, Gf = (T(t.float()) for t in (q, k, v, go))
        schf = J.Schedule(Qf)

        def step32(e=None):
            if e:
                e[0].record(stream)
            sv = J.jagged_flash_attention_forward(Qf, Kf, Vf, 64, 64, schedule=schf)
            if e:
                e[1].record(stream)
            J.jagged_flash_attention_backward(Qf, Kf, Vf, Gf, sv, schedule=schf)
            if e:
                e[2].record(stream)

        for _ in range(2):
            step32()
        ev32 = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(2)]
        for e in ev32:
            step32(e)
        torch.cuda.synchronize()
        f_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev32]))
        b_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev32]))
        fp32 = {"fwd_ms": f_ms, "bwd_ms": b_ms, "ms_per_step": f_ms + b_ms,
                "tflops": (fwd_fl + bwd_fl) / ((f_ms + b_ms) * 1e-3) / 1e12,
                "x_bf16_step": (f_ms + b_ms) / (elapsed_ms / args.steps),
                "path": "tcgen05 fp16 two-piece emulation (attn_x3_sm100.cu; JG_FP32_X3=1: bf16 three-piece), fp32 in/out, 2 timed steps"}
        del Qf, Kf, Vf, Gf, schf

    t = torch.tensor([elapsed_ms, e2e_s], dtype=torch.float64, device=dev)
    nb = torch.tensor([h2d, d2h], dtype=torch.float64, device=dev)  # whole-job copy bytes per step
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(nb, op=dist.ReduceOp.SUM)
    elapsed_ms, e2e_s = float(t[0]), float(t[1])
    h2d, d2h = float(nb[0]), float(nb[1])
    if rank != 0:
        return

    ms_per_step = elapsed_ms / args.steps
    value = (tot_fwd + tot_bwd) * args.steps / (elapsed_ms * 1e-3) / 1e12
    pk_burst, pk_sust, hbm, src = peaks()
    dominant = ("jagged_flash_attention_backward", bwd_fl, bwd_ms) if bwd_ms >= fwd_ms else \
        ("jagged_flash_attention_forward", fwd_fl, fwd_ms)
    achieved = dominant[1] / (dominant[2] * 1e-3) / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(dominant[0])
        except (ValueError, OSError):
            traffic = None
    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = cpu_reference_sample(lengths_all[:CFG["batch_per_gpu"]], H, D, target_s=args.cpu_seconds)
            cpu = {k2: cpu[k2] for k2 in ("value", "unit", "cores", "kind", "sample")}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "TFLOP/s", "cores": 0, "kind": "port", "sample": f"unavailable: {e}"}
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "cfg3: jagged flash attention fwd+bwd, B=1024 per GPU, max_len=1024, D=128, H=4, "
                               "half-mean lengths seed 0 (BASELINE.json configs[2])",
                   "global_batch": int(len(lengths_all)), "max_len": L, "head_dim": D, "heads": H,
                   "sum_B": int(lengths_all.sum()), "sum_sq_per_head": tot_sq,
                   "useful_flop_per_step": tot_fwd + tot_bwd, "parallelism": f"dp{world} (Bi^2-balanced sample shards)",
                   "l2": "inputs larger than L2 (537 MB per tensor at N=1)"},
        "roofline": {"bound": "tensor", "kernel": dominant[0], "achieved": achieved,
                     "peak": pk_burst, "unit": "TFLOP/s", "frac": achieved / pk_burst, "traffic": traffic,
                     "peak_source": f"{src} burst bf16 (MEASURED_PEAKS.json); sustained {pk_sust}",
                     "flop_per_launch": dominant[1], "ms_per_launch": dominant[2]},
        "step_ms_p10_p50_p90": [float(np.percentile(step_ms, q)) for q in (10, 50, 90)],
        "kernels": {"fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
                    "fwd_tflops": fwd_fl / (fwd_ms * 1e-3) / 1e12, "bwd_tflops": bwd_fl / (bwd_ms * 1e-3) / 1e12},
        "cpu_baseline": cpu,
        "e2e": {"value": (tot_fwd + tot_bwd) / e2e_s / 1e12 if e2e_s == e2e_s else None, "unit": "TFLOP/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_s * 1e3 if e2e_s == e2e_s else None,
                "api": "jg_jagged_flash_attention_fwd_bwd_host (pinned host buffers)"},
        "clocks": clk,
        "gpu_launches": launches,
    }
    if verify is not None:
        line["verify"] = verify
    if fp32 is not None:
        line["fp32_mode"] = fp32
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ secondary BASELINE configs
# `--config cfg1|cfg2|cfg4|cfg5|dense` prints one JSON line per measured operator group; cfg3 (the
# headline) is the default mode above. Times are CUDA events on the launching stream after warm-up,
# median over `--steps`; inputs are device-resident (cfg4/cfg5 inputs exceed L2).
def _events_time(fn, steps, warmup):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def _graph_time(fn, steps):
    """Device time of `fn` replayed from a captured CUDA graph (no host/launch overhead; small configs are
    launch-latency bound in eager mode). Returns ms, or None if capture is not possible."""
    import torch

    try:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()  # warm-up on the capture stream (one-time attribute setup happens outside the capture)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        g.replay()
        torch.cuda.synchronize()
        return _events_time(g.replay, steps, 2)
    except Exception as e:  # noqa: BLE001 — diagnostic leg only
        print(f"graph capture failed: {e}", file=sys.stderr)
        return None


def _cpu_ref_time(fn, reps=3):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def run_configs(args):
    import torch

    from paper_2409_15373_b200 import _lib, synth
    from paper_2409_15373_b200 import jagged as J

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    lib = _lib.lib()
    pk_burst, _, hbm, src = peaks()
    g = torch.Generator(device=dev).manual_seed(1)
    rnd = lambda *s, dt=torch.bfloat16: (torch.rand(*s, device=dev, generator=g) * 2 - 1).to(dt)  # noqa: E731
    kind, threads = _cpu_kind() if not args.no_cpu_baseline else ("none", 0)
    out = []

    def emit(line):
        line.setdefault("data", "synthetic")
        line.setdefault("n_gpus", 1)
        print(json.dumps(line), flush=True)
        out.append(line)

    cfg = args.config
    if cfg == "cfg1":
        # jagged_dense_bmm + jagged_softmax, B=64 L=128 D=64 T=32 uniform lengths seed 0, fp32
        ln = synth.gen_lengths("uniform", 128, 0, 64)
        off = synth.offsets_of(ln)
        S, B, D, T = int(off[-1]), 64, 64, 32
        X = J.JaggedTensor(torch.from_numpy(off).to(dev), rnd(S, D, dt=torch.float32), off)
        W = rnd(B, D, T, dt=torch.float32)

        def step():
            J.jagged_softmax(J.jagged_dense_bmm(X, W))

        ms = _events_time(step, args.steps, args.warmup)
        ms_graph = _graph_time(step, args.steps)
        eb = 4
        byts = (S * D + B * D * T + S * T) * eb + 2 * S * T * eb  # cost_model.cpp:153-155, :165-168
        flops = 2 * S * D * T
        cpu = None
        if kind != "none":
            from oracle import reference as F

            xh, wh = X.values.cpu().numpy(), W.cpu().numpy()
            t = _cpu_ref_time(lambda: F.jagged_softmax(off, F.jagged_dense_bmm(off, xh, wh, "f32", threads), "f32",
                                                       threads))
            cpu = {"value": byts / t / 1e9, "unit": "GB/s", "cores": threads, "kind": kind,
                   "sample": "full cfg1 (jagged_dense_bmm + jagged_softmax, fp32)", "us": t * 1e6}
        emit({"metric": "jagged-op GB/s", "config": {"workload": "cfg1: jagged_dense_bmm + jagged_softmax B=64 "
              "max_len=128 D=64 T=32 uniform seed 0", "sum_B": S}, "dtype": "f32", "value": byts / (ms * 1e-3) / 1e9,
              "unit": "GB/s", "us_per_step": ms * 1e3, "tflops": flops / (ms * 1e-3) / 1e12,
              "graph_us_per_step": ms_graph * 1e3 if ms_graph else None,
              "roofline": {"bound": "hbm", "achieved": byts / (ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                           "frac": byts / (ms * 1e-3) / 1e9 / hbm, "note": "~2.8 MB: launch-latency bound"},
              "cpu_baseline": cpu})
    elif cfg in ("cfg2", "cfg5"):
        if cfg == "cfg2":
            ln, D, H, fwd_only = synth.gen_lengths("zipf", 512, 0, 256, 1.1), 64, 1, True
            wl = "cfg2: JFA fwd B=256 max_len=512 D=64 H=1 bf16 Zipf(1.1) seed 0"
        else:
            ln, D, H, fwd_only = synth.gen_lengths("zipf", 4096, 0, 4096, 0.8), 128, 1, False
            wl = "cfg5: JFA fwd+bwd B=4096 max_len=4096 D=128 H=1 bf16 Zipf(0.8) seed 0"
        off = synth.offsets_of(ln)
        S = int(off[-1])
        Q, K, V, G = (J.JaggedTensor(torch.from_numpy(off).to(dev), rnd(S, H, D), off) for _ in range(4))
        sched = J.Schedule(Q)
        fwd_fl, bwd_fl, sq = useful_flops(ln, H, D)
        saved = J.jagged_flash_attention_forward(Q, K, V, schedule=sched)
        ms_f = _events_time(lambda: J.jagged_flash_attention_forward(Q, K, V, schedule=sched), args.steps, args.warmup)
        ms_fg = _graph_time(lambda: J.jagged_flash_attention_forward(Q, K, V, schedule=sched), args.steps)
        line = {"metric": "Jagged flash-attn " + ("fwd" if fwd_only else "fwd+bwd") + " TFLOP/s (useful FLOPs)",
                "config": {"workload": wl, "sum_B": S, "sum_sq": sq}, "dtype": "bf16",
                "fwd_ms": ms_f, "fwd_tflops": fwd_fl / (ms_f * 1e-3) / 1e12,
                "fwd_graph_ms": ms_fg, "fwd_graph_tflops": fwd_fl / (ms_fg * 1e-3) / 1e12 if ms_fg else None}
        total_fl, total_ms = fwd_fl, ms_f
        if not fwd_only:
            ws = torch.empty(J.backward_workspace_size(Q), dtype=torch.uint8, device=dev)
            ms_b = _events_time(lambda: J.jagged_flash_attention_backward(Q, K, V, G, saved, schedule=sched,
                                                                          workspace=ws), args.steps, args.warmup)
            line.update(bwd_ms=ms_b, bwd_tflops=bwd_fl / (ms_b * 1e-3) / 1e12)
            total_fl, total_ms = fwd_fl + bwd_fl, ms_f + ms_b
        line.update(value=total_fl / (total_ms * 1e-3) / 1e12, unit="TFLOP/s",
                    roofline={"bound": "tensor", "achieved": total_fl / (total_ms * 1e-3) / 1e12, "peak": pk_burst,
                              "unit": "TFLOP/s", "frac": total_fl / (total_ms * 1e-3) / 1e12 / pk_burst})
        if kind != "none":
            from oracle import reference as F

            stride = 1 if cfg == "cfg2" else 64
            sub = ln[::stride]
            sub = sub[sub > 0]
            so = synth.offsets_of(sub)
            ss = int(so[-1])
            r = np.random.default_rng(0)
            qh, kh, vh, gh = (r.uniform(-1, 1, (ss, D)).astype(np.float32) for _ in range(4))

            def cpu_run():
                o, l_ = F.jfa_forward(so, qh, kh, vh, 64, 64, "f32", threads)
                if not fwd_only:
                    F.jfa_backward(so, qh, kh, vh, gh, o, l_, 64, 64, "f32", threads)

            t = _cpu_ref_time(cpu_run, reps=1 if cfg == "cfg5" else 3)
            fl = (4 if fwd_only else 14) * D * int((sub * sub).sum())
            line["cpu_baseline"] = {"value": fl / t / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": kind,
                                    "sample": f"every {stride}th sample ({len(sub)} samples), fp32, {t:.1f} s"}
        emit(line)
    elif cfg == "cfg4":
        # jagged op suite at sum_B = 1,048,576 (half-mean B=2048 L=1024 seed 0), D=T=256, bf16 inputs
        ln = synth.gen_lengths("half-mean", 1024, 0, 2048)
        off = synth.offsets_of(ln)
        S, B, D = int(off[-1]), len(ln), 256
        sq = int((ln * ln).sum())
        X, Y = (J.JaggedTensor(torch.from_numpy(off).to(dev), rnd(S, D), off) for _ in range(2))
        A = J.Jagged2Tensor(X.offsets, rnd(sq), off)
        eb = 2
        ops = {
            "jagged_jagged_bmm_jagged_out": (lambda: J.jagged_jagged_bmm_jagged_out(X, Y), 2 * sq * D,
                                             (2 * S * D + sq) * eb),
            "array_jagged_bmm_jagged_out": (lambda: J.array_jagged_bmm_jagged_out(A, X), 2 * sq * D,
                                            (2 * S * D + sq) * eb),
            "jagged_jagged_bmm": (lambda: J.jagged_jagged_bmm(X, Y), 2 * S * D * D, (2 * S * D + B * D * D) * eb),
            "jagged_softmax": (lambda: J.jagged_softmax(X), 4 * S * D, 2 * S * D * eb),
            "jagged2_softmax": (lambda: J.jagged2_softmax(A), 4 * sq, 2 * sq * eb),
        }
        # the VJPs (linalg.cpp:283-507): bytes = inputs read + gradients written, flops = their contractions
        GX = J.JaggedTensor(X.offsets, rnd(S, D), off)
        GA = J.Jagged2Tensor(X.offsets, rnd(sq), off)
        GZ = rnd(B, D, D)
        ops.update({
            "jagged_jagged_bmm_jagged_out_vjp": (lambda: J.jagged_jagged_bmm_jagged_out_vjp(X, Y, GA), 4 * sq * D,
                                                 (4 * S * D + sq) * eb),
            "array_jagged_bmm_jagged_out_vjp": (lambda: J.array_jagged_bmm_jagged_out_vjp(A, X, GX), 4 * sq * D,
                                                (2 * sq + 3 * S * D) * eb),
            "jagged_jagged_bmm_vjp": (lambda: J.jagged_jagged_bmm_vjp(X, Y, GZ), 4 * S * D * D,
                                      (4 * S * D + B * D * D) * eb),
            "jagged_softmax_vjp": (lambda: J.jagged_softmax_vjp(X, GX), 6 * S * D, 3 * S * D * eb),
            "jagged2_softmax_vjp": (lambda: J.jagged2_softmax_vjp(A, GA), 6 * sq, 3 * sq * eb),
        })
        for name, (fn, fl, byts) in ops.items():
            ms = _events_time(fn, args.steps, args.warmup)
            gbs, tfs = byts / (ms * 1e-3) / 1e9, fl / (ms * 1e-3) / 1e12
            emit({"metric": "jagged-op GB/s", "op": name, "config": {"workload": "cfg4: half-mean B=2048 L=1024 "
                  "seed 0 (sum_B=1,048,576), D=T=256, bf16 in / bf16 out", "sum_sq": sq}, "dtype": "bf16",
                  "value": gbs, "unit": "GB/s", "ms": ms, "tflops": tfs,
                  "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                               "tensor_frac": tfs / pk_burst}})
    elif cfg == "dense":
        # the paper's jagged-vs-padded comparison on cfg3: padded dense attention (materialised masked
        # scores, PyTorch bf16 matmul + softmax, the paper's "PyTorch" column) and padded dense flash
        # attention (torch SDPA with a key-padding mask) vs our jagged flash attention, fwd+bwd, with
        # peak memory. These comparators are library code used only as baselines.
        ln = synth.gen_lengths(CFG["dist"], CFG["max_len"], CFG["seed"], CFG["batch_per_gpu"])
        off = synth.offsets_of(ln)
        S, B, L, D, H = int(off[-1]), len(ln), CFG["max_len"], CFG["head_dim"], CFG["heads"]
        fwd_fl, bwd_fl, _ = useful_flops(ln, H, D)
        Q, K, V, G = (J.JaggedTensor(torch.from_numpy(off).to(dev), rnd(S, H, D), off) for _ in range(4))
        sched = J.Schedule(Q)
        ws = torch.empty(J.backward_workspace_size(Q), dtype=torch.uint8, device=dev)

        def jagged_step():
            s_ = J.jagged_flash_attention_forward(Q, K, V, schedule=sched)
            J.jagged_flash_attention_backward(Q, K, V, G, s_, schedule=sched, workspace=ws)

        def measure(fn):
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats()
            base = torch.cuda.memory_allocated()
            ms = _events_time(fn, max(2, args.steps // 2), 2)
            return ms, (torch.cuda.max_memory_allocated() - base) / 2**30

        ms_j, mem_j = measure(jagged_step)
        # padded inputs [B, H, L, D] built from the same jagged values (jagged_to_dense on device)
        pad_blhd = lambda t: J.jagged_to_dense(J.JaggedTensor(t.offsets, t.values.reshape(S, H * D), off), L,  # noqa
                                               0.0).reshape(B, L, H, D)
        qd, kd, vd, gd = pad_blhd(Q), pad_blhd(K), pad_blhd(V), pad_blhd(G)
        qp, kp, vp, gp = (t.transpose(1, 2).contiguous() for t in (qd, kd, vd, gd))  # [B, H, L, D] for torch
        lens = torch.from_numpy(ln).to(dev)
        keymask = torch.arange(L, device=dev)[None, :] < lens[:, None]  # [B, L]
        addmask = torch.zeros(B, 1, 1, L, device=dev, dtype=torch.bfloat16).masked_fill(~keymask[:, None, None, :],
                                                                                          float("-inf"))

        def dense_step():
            q_, k_, v_ = (t.detach().requires_grad_() for t in (qp, kp, vp))
            s_ = torch.matmul(q_, k_.transpose(-1, -2)) * (D ** -0.5) + addmask
            p_ = torch.nan_to_num(torch.softmax(s_.float(), dim=-1), 0.0).to(torch.bfloat16)  # empty samples
            o_ = torch.matmul(p_, v_)
            o_.backward(gp)

        def flash_step():
            q_, k_, v_ = (t.detach().requires_grad_() for t in (qp, kp, vp))
            o_ = torch.nn.functional.scaled_dot_product_attention(q_, k_, v_, attn_mask=keymask[:, None, None, :])
            o_.backward(gp)

        ws_p = torch.empty(lib.jg_attention_backward_workspace_size(B * L, B, H, D), dtype=torch.uint8, device=dev)

        def padded_ours_step():  # the same kernels in padded mode (full L^2 work, masks)
            s_ = J.dense_flash_attention(qd, kd, vd, ln)
            J.dense_flash_attention_backward(qd, kd, vd, gd, s_, ln, workspace=ws_p)

        res = {"jagged_flash (ours)": (ms_j, mem_j)}
        for name, fn in (("padded dense flash (ours: same kernels, padded mode)", padded_ours_step),("padded dense attention (torch matmul+softmax)", dense_step),
                         ("padded dense flash (torch SDPA + mask)", flash_step)):
            try:
                res[name] = measure(fn)
            except RuntimeError as e:  # OOM on the padded baselines is itself the memory claim
                res[name] = (float("nan"), float("nan"))
                print(f"{name}: {e}", file=sys.stderr)
            torch.cuda.empty_cache()
        emit({"metric": "jagged vs padded attention fwd+bwd (cfg3)", "config": {"workload": "cfg3 B=1024 L=1024 D=128 "
              "H=4 bf16 half-mean seed 0", "padded_flops_ratio": float(B * L * L / (ln.astype(np.int64) ** 2).sum())},
              "dtype": "bf16", "value": ms_j, "unit": "ms",
              "results": {k2: {"ms": v2[0], "peak_GiB": v2[1], "useful_tflops": (fwd_fl + bwd_fl) / (v2[0] * 1e-3) / 1e12}
                          for k2, v2 in res.items()},
              "speedup_vs_dense": res["padded dense attention (torch matmul+softmax)"][0] / ms_j,
              "speedup_vs_dense_flash": res["padded dense flash (torch SDPA + mask)"][0] / ms_j,
              "speedup_vs_padded_same_kernels": res["padded dense flash (ours: same kernels, padded mode)"][0] / ms_j,
              "memory_ratio_vs_padded_same_kernels": res["padded dense flash (ours: same kernels, padded mode)"][1] / mem_j,
              "memory_ratio_vs_dense": res["padded dense attention (torch matmul+softmax)"][1] / mem_j,
              "memory_ratio_vs_dense_flash": res["padded dense flash (torch SDPA + mask)"][1] / mem_j})
    elif cfg == "table1":
        run_table1(args, J, synth, dev, rnd, emit)
    if args.out:
        with open(args.out, "a") as f:
            for line in out:
                f.write(json.dumps(line) + "\n")


def run_table1(args, J, synth, dev, rnd, emit):
    """the reference bench's records (bench.hpp:61-81, bench.cpp:200-372) for the GPU variants.
    Per Table-1 op: variants[0] = "padded" (the same op on padded tensors with torch bf16 kernels — library
    baseline), "jagged" = ours; the attention sweep point has the reference's four variants (dense_attention:
    torch padded matmul+softmax; dense_flash_attention: our kernels in padded mode; jagged_attention /
    jagged_flash_attention: ours). Outputs are cross-checked on the valid region before timing (bf16: max-abs
    error <= 2e-2 x max|ref|), times are CUDA-event p10/p50/p90 over --steps, FLOPs/bytes come from the
    reference's cost model (report.py), and the report is written in the reference's csv/json/md formats."""
    import torch

    from paper_2409_15373_b200 import report as RP

    B, L, D, T, seed = 1024, 1024, 128, 128, 0
    ln = synth.gen_lengths("half-mean", L, seed, B)
    off = synth.offsets_of(ln)
    S, sq = int(off[-1]), int((ln * ln).sum())
    offd, lens = torch.from_numpy(off).to(dev), torch.from_numpy(ln).to(dev)
    rowmask = torch.arange(L, device=dev)[None, :] < lens[:, None]  # [B, L]
    sqmask = rowmask[:, :, None] & rowmask[:, None, :]              # [B, L, L]
    jt = lambda v: J.JaggedTensor(offd, v, off)  # noqa: E731
    X, K2, Y = jt(rnd(S, D)), jt(rnd(S, D)), jt(rnd(S, T))
    A = J.Jagged2Tensor(offd, rnd(sq), off)
    Wd = rnd(B, D, T)
    W0, b0, W1, b1 = rnd(D, T) * D ** -0.5, rnd(T) * 0.1, rnd(T, D) * T ** -0.5, rnd(D) * 0.1
    layers = [J.MlpLayer(W0, b0, J.RELU), J.MlpLayer(W1, b1, J.NONE)]
    Xp, K2p, Yp, Ap = J.jagged_to_dense(X, L), J.jagged_to_dense(K2, L), J.jagged_to_dense(Y, L), J.jagged2_to_dense(A, L)
    ninf = float("-inf")

    def times_us(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        return ts

    def crosscheck(op, got, ref):
        g, r = got.float(), ref.float()
        err = float((g - r).abs().max()) if r.numel() else 0.0
        scale = max(float(r.abs().max()) if r.numel() else 0.0, 1e-30)
        if not err <= 2e-2 * scale:
            raise RuntimeError(f"{op}: jagged/padded outputs diverge before timing: max abs err {err:.3e} "
                               f"vs 2e-2 x max|ref| {scale:.3e}")
        return float(g.double().sum())

    records = []

    def record(op, variants, T_=T):
        """variants: [(name, fn, valid_region_of_output)], [0] the padded baseline."""
        ref_valid = variants[0][2](variants[0][1]())
        rec = RP.BenchRecord(op, B, D, T_, L, "half_mean", seed, "bf16", 1)
        for name, fn, valid in variants:
            cs = crosscheck(op, valid(fn()), ref_valid)
            rec.variants.append(RP.VariantStats.from_times(name, times_us(fn), cs))
        rec.finalize(RP.OpConfig(op, D, T_, list(ln), 2, L))
        records.append(rec)

    rows = lambda t: t[rowmask]  # noqa: E731  padded [B, L, C] -> the jagged rows
    vals = lambda t: t.values  # noqa: E731
    record("jagged_dense_bmm", [("padded", lambda: torch.bmm(Xp, Wd), rows),
                                ("jagged", lambda: J.jagged_dense_bmm(X, Wd), vals)])
    record("jagged_jagged_bmm", [("padded", lambda: torch.bmm(Xp.transpose(1, 2), Yp), lambda t: t),
                                 ("jagged", lambda: J.jagged_jagged_bmm(X, Y), lambda t: t)])
    record("jagged_softmax", [("padded", lambda: torch.softmax(Xp.masked_fill(~rowmask[:, :, None], ninf), dim=1)
                               .nan_to_num_(0.0), rows), ("jagged", lambda: J.jagged_softmax(X), vals)], T_=1)
    record("jagged_jagged_bmm_jagged_out", [("padded", lambda: torch.bmm(Xp, K2p.transpose(1, 2)), lambda t: t[sqmask]),
                                            ("jagged", lambda: J.jagged_jagged_bmm_jagged_out(X, K2), vals)], T_=1)
    record("array_jagged_bmm_jagged_out", [("padded", lambda: torch.bmm(Ap, Xp), rows),
                                           ("jagged", lambda: J.array_jagged_bmm_jagged_out(A, X), vals)], T_=1)
    record("jagged2_softmax", [("padded", lambda: torch.softmax(Ap.masked_fill(~sqmask, ninf), dim=2).nan_to_num_(0.0),
                                lambda t: t[sqmask]), ("jagged", lambda: J.jagged2_softmax(A), vals)], T_=1)

    def mlp_padded():
        h = torch.relu(torch.addmm(b0, Xp.reshape(B * L, D), W0))
        return torch.addmm(b1, h, W1).reshape(B, L, D)

    record("jagged_mlp", [("padded", mlp_padded, rows), ("jagged", lambda: J.jagged_mlp(X, layers), vals)])

    # the attention sweep point (bench.cpp:317-372, 476-503): one record per variant, ratios vs dense_attention
    Q1, K1, V1 = (jt(rnd(S, 1, D)) for _ in range(3))
    Qp, Kp, Vp = (J.jagged_to_dense(J.JaggedTensor(offd, t.values.reshape(S, D), off), L) for t in (Q1, K1, V1))
    keymask = sqmask

    def dense_attention():
        s_ = torch.bmm(Qp, Kp.transpose(1, 2)) * D ** -0.5
        p_ = torch.softmax(s_.masked_fill(~keymask, ninf), dim=-1).nan_to_num_(0.0)
        return torch.bmm(p_, Vp)

    att = [("dense_attention", dense_attention, rows),
           ("dense_flash_attention", lambda: J.dense_flash_attention(Qp, Kp, Vp, ln).output, rows),
           ("jagged_attention", lambda: J.jagged_attention(Q1, K1, V1), lambda t: t.values.reshape(S, D)),
           ("jagged_flash_attention", lambda: J.jagged_flash_attention_forward(Q1, K1, V1).output,
            lambda t: t.values.reshape(S, D))]
    ref_valid = rows(dense_attention())
    stats = []
    for name, fn, valid in att:
        cs = crosscheck("attention", valid(fn()), ref_valid)
        stats.append(RP.VariantStats.from_times(name, times_us(fn), cs))
    cfg_a = RP.OpConfig("jagged_flash_attention", D, 1, list(ln), 2, L)
    dense_bytes = RP.variant_bytes(cfg_a, "dense_attention")
    for st_ in stats:
        rec = RP.BenchRecord("attention", B, D, 1, L, "half_mean", seed, "bf16", 1)
        c = RP.OpConfig(st_.variant, D, 1, list(ln), 2, L)
        rec.flops_jagged, rec.flops_padded = RP.flops_of(c)
        rec.bytes_jagged, rec.bytes_padded = RP.bytes_of(c)
        st_.flops, st_.bytes = RP.variant_flops(c, st_.variant), RP.variant_bytes(c, st_.variant)
        st_.speedup_vs_dense = stats[0].time_us_p50 / st_.time_us_p50
        st_.bytes_ratio_vs_dense = st_.bytes / dense_bytes
        rec.variants = [st_]
        records.append(rec)
    for r in records:
        emit({"metric": "table1 record (reference bench schema)", "config": {"workload": f"half-mean B={B} L={L} "
              f"seed {seed}, D={D}, T={T}, bf16, {args.steps} timed iterations"}, "dtype": "bf16",
              "record": json.loads(RP.render_report([r], "json"))[0]})
    if args.report:
        for fmt in ("csv", "json", "md"):
            with open(f"{args.report}.{fmt}", "w") as f:
                f.write(RP.render_report(records, fmt))


def _free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return int(so.getsockname()[1])


def relaunch_ranks(n: int) -> int:
    """`--gpus N` (N > 1) outside torchrun: re-run this script as N ranks through torch.distributed.run on one
    node (rendezvous on 127.0.0.1), so `python bench.py --gpus N` is a real N-rank run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {n} ranks: {' '.join(cmd[2:6])} ...", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def selftest_launch(rank: int, world: int) -> None:
    """--selftest-launch: the rank plumbing alone on CPU (gloo): every rank joins, one all-reduce, rank 0 reports."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"selftest": "launch", "n_ranks": dist.get_world_size(), "rank_sum": float(t.item()),
                          "backend": dist.get_backend()}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=30.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32-mode leg (profiling runs)")
    ap.add_argument("--config", default="cfg3", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "dense", "table1"],
                    help="cfg3 = the headline JSON line; the others measure the secondary BASELINE configs")
    ap.add_argument("--out", default=None, help="also append secondary-config lines to this file")
    ap.add_argument("--report", default=None,
                    help="--config table1: write the records as PATH.csv / PATH.json / PATH.md (reference formats)")
    ap.add_argument("--selftest-launch", action="store_true", help=argparse.SUPPRESS)  # CPU test of the rank launch
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_ranks(args.gpus))
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.gpus else 1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ:
        world = 1  # single process
    if args.selftest_launch:
        selftest_launch(rank, world)
        return
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if args.config != "cfg3":
        run_configs(args)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
