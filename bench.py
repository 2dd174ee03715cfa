#!/usr/bin/env python
"""Benchmark: Jagged Flash Attention fwd+bwd, useful TFLOP/s (BASELINE.json configs[2] = "cfg3").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step = one jagged_flash_attention_forward + jagged_flash_attention_backward over the rank's
shard of the batch (B=1024 per GPU, max_len=1024, D=128, H=4, bf16, half-mean lengths seed 0).
Useful FLOPs = 14·H·D·ΣBi² per step (fwd 4·H·D·ΣBi², bwd 10·H·D·ΣBi²; padding never counted).
Weak scaling: the global batch is 1024·N samples, sharded on Bi²-balanced sample boundaries, no
collective inside the timed region. Inputs (537 MB per tensor) are larger than L2.

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
    ws = torch.empty(lib.jg_attention_backward_workspace_size(S, H, D), dtype=torch.uint8, device=dev)
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

    t = torch.tensor([elapsed_ms, e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms, e2e_s = float(t[0]), float(t[1])
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
        "kernels": {"fwd_ms": fwd_ms, "bwd_ms": bwd_ms,
                    "fwd_tflops": fwd_fl / (fwd_ms * 1e-3) / 1e12, "bwd_tflops": bwd_fl / (bwd_ms * 1e-3) / 1e12},
        "cpu_baseline": cpu,
        "e2e": {"value": (tot_fwd + tot_bwd) / e2e_s / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3,
                "api": "jg_jagged_flash_attention_fwd_bwd_host (pinned host buffers)"},
        "clocks": clk,
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.gpus else 1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ:
        world = 1  # single process
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
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
