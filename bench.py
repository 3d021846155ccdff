#!/usr/bin/env python
"""bench.py — exact top-k decode attention, µs per layer decode step (BASELINE.json metric).

Workload (N=1 default): BASELINE cfg3 — one layer, Llama-3-8B head shape (Hq=32, Hkv=8,
d=128), N = 1,048,576 context rows, k = 16,384 per q head (1.6 %), batch 1, bf16 K/V cache,
i.i.d. standard-normal synthetic data (the reference's own distribution, bench.py:335-342).
The K cache (2.15 GB) is far larger than L2 (126 MB), so every step streams it from HBM;
no L2 flush is needed between steps.

  value     µs per layer-step, inputs resident in HBM, CUDA events over K steps
  e2e       same metric through TopkDecoder.step() -> (out, idx) with pinned HOST buffers:
            q and the new token's k/v rows read from host memory, KV append, attention, out and
            the selected ids back in host memory, every step (the whole device part replayed as
            one CUDA graph; the host syncs on the result each step); `out_only` = same without ids
  roofline  dominant kernel (key scan): algorithmic K bytes / scan-kernel time (events
            recorded around the scan launch on its stream, every timed step)
  cpu_baseline  the reference algorithm's C port (oracle/) on the host cores: one full
            layer-step on every host thread, plus a single-core sample (1 KV group, scaled)

Multi-GPU (torchrun, N > 1): the context is sharded by token range (strong scaling: the 1M
rows are split across ranks); value = max over ranks of the per-step device time. Default
exchange (`--exchange symm`): every rank publishes its narrow (top ~ceil(1.5*k/N)) and full
candidate lists in torch symmetric memory, the merge kernel reads the peers' lists over NVLink
and picks narrow or full per head on the device, the finishing kernel sums the peers' partials
(DeviceShardedStep: no host round trip). `--exchange nccl`: all-gather + all-reduce through
NCCL collectives (sharded_topk_attention, one host read of the exactness flag per step).
`--impl reference`: times the reference algorithm's CPU port on rank 0 (others exit 0).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HQ, HKV, D = 32, 8, 128
CONFIGS = {
    "cfg1": dict(B=1, N=16384, k=256),
    "cfg2": dict(B=1, N=131072, k=2048),
    "cfg3": dict(B=1, N=1 << 20, k=16384),
    "cfg5": dict(B=16, N=262144, k=4096),
    # one rank's shard of cfg3 at 8 GPUs (its local top-k over 131,072 rows): diagnostics only
    "cfg3_g8": dict(B=1, N=131072, k=16384),
}
METRIC = "us_per_layer_decode_step"
WINDOW_CAP = 256


def algo_bytes(B, N, k):
    """K scan + selected V rows + q in/out + int32 ids, per layer-step."""
    return B * N * HKV * D * 2 + B * HQ * k * D * 2 + B * HQ * D * 2 * 2 + B * HQ * k * 4


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# the dominant kernel: the TMA + tcgen05 key scan unless TKV_SCAN=hmma selects the mma.sync scan
SCAN_KERNEL = "scan_kernel" if os.environ.get("TKV_SCAN", "") == "hmma" else "scan_tc_kernel"
SCAN_DESC = {"scan_kernel": "scan_kernel (mma.sync GQA key scan + candidate emit)",
             "scan_tc_kernel": "scan_tc_kernel (TMA + tcgen05 GQA key scan + candidate emit)"}


def scan_traffic(config: str, world: int):
    """dram__bytes_read.sum + dram__bytes_write.sum of the scan kernel per launch, from the
    committed ncu --set full capture (profiles/r*_summary.json); None when not captured."""
    if config != "cfg3" or world != 1:
        return None
    caps = sorted((ROOT / "profiles").glob("r*_summary.json"))
    if not caps:
        return None
    j = json.loads(caps[-1].read_text())
    return j.get(SCAN_KERNEL, {}).get("traffic_bytes")


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle-reason sampling (NVML) during the timed region."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover
            self.error = str(e)
        return self

    def _run(self):
        nv = self._nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for n, bit in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def make_inputs(cfg, rows, seed, device, rank_lo=0, rank_hi=None):
    """Seeded standard-normal bf16 K/V/q generated on the device (same values for every
    sharding: each rank generates the full-row stream of its range by chunked seeds)."""
    import torch

    B, N = cfg["B"], cfg["N"]
    hi = N if rank_hi is None else rank_hi
    n = hi - rank_lo
    K = torch.zeros((B, HKV, rows, D), dtype=torch.bfloat16, device=device)
    V = torch.zeros((B, HKV, rows, D), dtype=torch.bfloat16, device=device)
    chunk = 8192
    for c0 in range(0, N, chunk):
        c1 = min(N, c0 + chunk)
        lo, hi2 = max(c0, rank_lo), min(c1, hi)
        if lo >= hi2:
            continue
        g = torch.Generator(device=device).manual_seed(seed * 1000003 + c0)
        blk = torch.randn((2, B, HKV, c1 - c0, D), generator=g, device=device).to(torch.bfloat16)
        K[:, :, lo - rank_lo:hi2 - rank_lo] = blk[0, :, :, lo - c0:hi2 - c0]
        V[:, :, lo - rank_lo:hi2 - rank_lo] = blk[1, :, :, lo - c0:hi2 - c0]
    g = torch.Generator(device=device).manual_seed(seed * 7919 + 1)
    q = torch.randn((B, HQ, D), generator=g, device=device).to(torch.bfloat16)
    return q, K, V, n


def _cpu_inputs(cfg, kv_groups: int, seed: int = 1234):
    """Standard-normal K/V/q rounded to bf16 values (what the GPU arm sees), f32 storage,
    generated in row chunks so the 1M-row cache needs no f64 temporaries."""
    import numpy as np

    from oracle import oracle as O

    B, N = cfg["B"], cfg["N"]
    G = HQ // HKV
    rng = np.random.default_rng(seed)
    K = np.empty((B, kv_groups, N, D), dtype=np.float32)
    V = np.empty_like(K)
    step = 1 << 16
    for b in range(B):
        for g in range(kv_groups):
            for r0 in range(0, N, step):
                r1 = min(N, r0 + step)
                K[b, g, r0:r1] = O.to_bf16_f32(rng.standard_normal((r1 - r0, D), dtype=np.float32))
                V[b, g, r0:r1] = O.to_bf16_f32(rng.standard_normal((r1 - r0, D), dtype=np.float32))
    q = O.to_bf16_f32(rng.standard_normal((B, kv_groups * G, D), dtype=np.float32))
    return q, K, V


def _time_port(q, K, V, N, k, threads, reps_budget_s, max_reps):
    """Repeated oracle/tkv_oracle.c layer calls; returns the per-call seconds."""
    from oracle import oracle as O

    times = []
    t_end = time.perf_counter() + reps_budget_s
    while not times or (time.perf_counter() < t_end and len(times) < max_reps):
        t0 = time.perf_counter()
        O.c_decode_layer(q, K, V, [N] * q.shape[0], k, threads=threads)
        times.append(time.perf_counter() - t0)
    return times


PORT_DESC = ("oracle/tkv_oracle.c (C port of ann_kernels.py:31-47, ann.py:154-167, "
             "attention.py:107-167: strict left-to-right f64 scan, _flat_topk, f64 joint softmax)")


def cpu_baseline(cfg, seconds_budget=20.0):
    """The reference algorithm's CPU port on the host cores (test infrastructure, timed as the
    baseline): ONE FULL layer-step of the workload (every KV group and batch entry, all Hq
    heads, all host threads), plus a single-core sample of one KV group (scaled to a layer-step
    and labelled as such) for the per-core comparison BASELINE.md §3 plans."""
    from oracle import oracle as O

    N, k, B = cfg["N"], cfg["k"], cfg["B"]
    t = int(O.c_lib().tkv_oracle_max_threads())
    q, K, V = _cpu_inputs(cfg, HKV)
    full = _time_port(q, K, V, N, k, t, seconds_budget / 2, 3)
    G = HQ // HKV
    one = _time_port(q[:1, :G].copy(), K[:1, :1], V[:1, :1], N, k, 1, seconds_budget / 4, 2)
    return {"value": round(min(full) * 1e6, 1), "unit": "us", "cores": t, "kind": "port",
            "sample": f"full layer-step (B={B}, Hq={HQ}, Hkv={HKV}, N={N}, k={k}) through {PORT_DESC}, "
                      f"{t} OpenMP threads (one head per thread), best of {len(full)}",
            "single_core": {"value": round(min(one) * HKV * B * 1e6, 1), "unit": "us", "cores": 1,
                            "sample": f"1 KV group ({G} q heads) of 1 batch entry on 1 thread, best of "
                                      f"{len(one)}, scaled x{HKV * B} to one layer-step"}}


L2_BYTES = 126 * 1024 * 1024


def layer_caches(cfg, world=1):
    """How many independent layer caches (K, V, q) the timed steps cycle through, as the layers
    of a model do: enough that the K bytes streamed between two uses of one cache are >= 4x L2,
    so no step finds its keys or its selected V rows in L2 (cfg1: 16, cfg2: 2, cfg3: 1)."""
    kb = cfg["B"] * cfg["N"] * HKV * D * 2 / world
    return max(1, math.ceil(4 * L2_BYTES / kb))


def our_config(args, cfg, world=1):
    B, N, k = cfg["B"], cfg["N"], cfg["k"]
    kgb = B * N * HKV * D * 2 / world / 1e9
    R = layer_caches(cfg, world)
    l2 = ("inputs larger than L2 (K cache %.2f GB per GPU, L2 126 MB): no flush" % kgb if R == 1 else
          "%d independent layer caches cycled step by step (K %.3f GB each per GPU; %.2f GB of keys between "
          "two uses of one cache, > 4x the 126 MB L2): no flush" % (R, kgb, R * kgb))
    c = {"workload": args.config, "batch": B, "n_ctx": N, "k": k, "Hq": HQ, "Hkv": HKV, "head_dim": D,
         "parallelism": f"token-shard{world}" if world > 1 else "single",
         "l2": l2, "seed": args.seed}
    if world > 1 and args.narrow:
        c["narrow_c"] = args.narrow
    if world > 1:
        c["exchange"] = ("device-driven, torch symmetric memory (DeviceShardedStep)" if args.exchange == "symm"
                         else "NCCL all-gather + all-reduce (sharded_topk_attention)")
    return c


def run_reference(args, cfg):
    """--impl reference: the reference's algorithm on the host CPU (its CPU port; the reference
    itself is Python/Numba with no compiled sources to build), timed on exactly
    this arm's workload: every step is one FULL layer-step, repeated for up to ~2 minutes."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O

    N, k, B = cfg["N"], cfg["k"], cfg["B"]
    t = int(O.c_lib().tkv_oracle_max_threads())
    q, K, V = _cpu_inputs(cfg, HKV)
    # warm-up (page in the caches, OpenMP pool), then the timed steps
    warm = _time_port(q, K, V, N, k, t, 0.0, 1)
    per = warm[0]
    steps = max(1, min(args.steps, int(120.0 / max(per, 1e-3))))
    times = _time_port(q, K, V, N, k, t, 1e9, steps)
    us = sum(times) / len(times) * 1e6
    cb = {"value": round(us, 1), "unit": "us", "cores": t, "kind": "port",
          "sample": f"{len(times)} full layer-steps (B={B}, Hq={HQ}, Hkv={HKV}, N={N}, k={k}) through {PORT_DESC}, "
                    f"{t} OpenMP threads, mean"}
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "us",
            "n_gpus": args.gpus, "steps": len(times), "steps_requested": args.steps, "warmup": 1,
            "ms_per_step": round(us / 1e3, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": our_config(args, cfg, 1), "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--exchange", default="symm", choices=["symm", "nccl"],
                    help="N>1: device-driven exchange over torch symmetric memory (DeviceShardedStep; "
                         "falls back to nccl when unavailable) or NCCL collectives (sharded_topk_attention)")
    ap.add_argument("--narrow", type=float, default=1.5,
                    help="N>1: narrow candidate exchange, each rank sends its top ceil(C*k/N) "
                         "(exactness checked per step, full-k fallback); 0 = full-k exchange")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_2502_06766_b200 as tkv
    from paper_2502_06766_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _lib.check(_lib.load().tkv_device_check())
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    B, N, k = cfg["B"], cfg["N"], cfg["k"]
    steps, warm = args.steps, args.warmup

    lo, hi = tkv.shard_range(N, world, rank)
    rows = (hi - lo) + WINDOW_CAP
    R = layer_caches(cfg, world)
    reps = [make_inputs(cfg, rows, args.seed + r, dev, lo, hi) for r in range(R)]
    q, K, V, n_local = reps[0]
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)

    scan_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in scan_ev:  # torch creates the cudaEvent_t lazily, on first record
        a.record(stream)
        b.record(stream)
    lib = _lib.load()

    if world == 1:
        out = torch.empty((B, HQ, D), dtype=torch.float32, device=dev)
        idx = torch.empty((B, HQ, k), dtype=torch.int32, device=dev)
        sc = torch.empty((B, HQ, k), dtype=torch.float32, device=dev)
        n_ctx = torch.full((B,), n_local, dtype=torch.int32, device=dev)
        prob = tkv.ops.make_problem(B, HQ, HKV, rows, n_local, k)
        ws = tkv.Workspace(prob, dev)

        def step(i=0):
            qr, Kr, Vr, _ = reps[i % R]
            tkv.topk_decode_attention(qr, Kr, Vr, n_ctx, k, out=out, idx=idx, scores=sc, workspace=ws,
                                      max_ctx=n_local)
    else:
        stages = tkv.CudaStages(B, HQ, HKV, rows, n_local, k, row_offset=lo, device=dev)
        n_ctx = torch.full((B,), n_local, dtype=torch.int32, device=dev)
        kk = tkv.narrow_k(k, world, args.narrow) if args.narrow else k
        step = None
        if args.exchange == "symm":
            try:
                exch = tkv.SymmetricExchange(B, HQ, k, kk, dev)
                dstep = tkv.DeviceShardedStep(stages, exch, rank, kk)
                n_win0 = torch.zeros(B, dtype=torch.int32, device=dev)

                def step(i=0):
                    qr, Kr, Vr, _ = reps[i % R]
                    dstep(qr, Kr, Vr, n_ctx, n_win0)
            except Exception as e:  # pragma: no cover - depends on the node's symmetric memory support
                print(f"[bench] symmetric-memory exchange unavailable ({e!r}); using NCCL collectives",
                      file=sys.stderr)
                args.exchange = "nccl"
        if step is None:
            gathered = torch.empty(world * B * HQ * k, dtype=torch.int64, device=dev)
            narrow = None
            if args.narrow:
                narrow = tkv.CudaStages(B, HQ, HKV, rows, n_local, kk, row_offset=lo, device=dev)

            def step(i=0):
                qr, Kr, Vr, _ = reps[i % R]
                tkv.sharded_topk_attention(stages, qr, Kr, Vr, n_ctx, None, gathered=gathered,
                                           narrow=narrow)

    for i in range(warm):
        step(i)
    launches_per_step = _lib.launches() if world == 1 else None
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # the K timed steps run exactly as a user's calls do (no profiling hooks in the stream,
        # so the kernels keep their programmatic dependent launches)
        e0.record(stream)
        for i in range(steps):
            step(i)
        e1.record(stream)
        torch.cuda.synchronize()
        # the dominant kernel's duration: the same steps again, CUDA events recorded by the
        # library around the key-scan launch on its stream
        for i in range(steps):
            lib.tkv_profile_scan_events(scan_ev[i][0].cuda_event, scan_ev[i][1].cuda_event)
            step(i)
        torch.cuda.synchronize()
    lib.tkv_profile_scan_events(None, None)
    ms = e0.elapsed_time(e1) / steps
    scan_ms = sum(a.elapsed_time(b) for a, b in scan_ev) / steps
    if world > 1:
        t = torch.tensor([ms, scan_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, scan_ms = t.tolist()
        dist.barrier()
    if world == 1:
        launches_per_step = _lib.launches()

    # ---------------- e2e through the public decode API with host buffers (N = 1)
    e2e = None
    if world == 1:
        decs = [tkv.TopkDecoder(Kr, Vr, n_local, k, max_ctx=n_local) for _, Kr, Vr, _ in reps]
        qh = q.cpu().pin_memory()
        kn = torch.randn((B, HKV, D)).to(torch.bfloat16).pin_memory()
        vn = torch.randn((B, HKV, D)).to(torch.bfloat16).pin_memory()
        e2e_steps = max(1, min(steps, (WINDOW_CAP - 2 * max(warm, R) - 2) // 2))

        def e2e_run(return_idx):
            for i in range(max(warm, R)):  # every cache's decoder: graph upload before timing
                decs[i % R].step(qh, kn, vn, return_idx=return_idx)
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for i in range(e2e_steps):
                decs[i % R].step(qh, kn, vn, return_idx=return_idx)
            a1.record(stream)
            torch.cuda.synchronize()
            return a0.elapsed_time(a1) / e2e_steps * 1e3

        e2e_idx_us = e2e_run(True)
        e2e_out_us = e2e_run(False)
        h2d = qh.numel() * 2 + kn.numel() * 2 + vn.numel() * 2
        e2e = {"value": round(e2e_idx_us, 2), "unit": "us", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": B * HQ * D * 4 + B * HQ * k * 4, "steps": e2e_steps,
               "path": "TopkDecoder.step(q, k_new, v_new) -> (out, idx) with pinned host tensors: CUDA-graph "
                       "replay (a staging kernel reads q/k/v in place from pinned host memory, KV append, "
                       "top-k attention writing out and the selected ids straight into pinned host memory) "
                       "-> host sync, every step",
               "out_only": {"value": round(e2e_out_us, 2), "d2h_bytes_per_step": B * HQ * D * 4,
                            "path": "the same step with return_idx=False (ids stay on the device)"}}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peak, peak_kind = peaks()
    kbytes = B * (hi - lo) * HKV * D * 2
    achieved = kbytes / (scan_ms * 1e-3) / 1e9
    step_bytes = algo_bytes(B, N, k) / world
    cb = None
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(cfg)
    line = {
        "metric": METRIC, "value": round(ms * 1e3, 2), "unit": "us", "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": round(ms, 5), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": our_config(args, cfg, world),
        "roofline": {"bound": "hbm", "kernel": SCAN_DESC[SCAN_KERNEL],
                     "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": scan_traffic(args.config, world),
                     "algorithmic_bytes_per_launch": kbytes, "kernel_us": round(scan_ms * 1e3, 2)},
        "step_roofline": {"algorithmic_bytes": int(step_bytes),
                          "achieved_gbs": round(step_bytes / (ms * 1e-3) / 1e9, 1),
                          "frac": round(step_bytes / (ms * 1e-3) / 1e9 / peak, 4)},
        "cpu_baseline": cb,
        "e2e": e2e,
        "gpu_launches": (launches_per_step or 0) * steps if world == 1 else None,
        "clocks": clk.summary(),
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
