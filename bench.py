#!/usr/bin/env python3
"""Benchmark: fp64 GFLOP/s of the tuned kernels on B200 (BASELINE.json metric).

Headline workload (configs[1]): LU without pivoting, PolyBench LARGE N=2000,
fixed block (by, bx) = BENCH_LU_BLOCK, inputs gen_spd(2000, seed=1).  A step
is one in-place factorisation of one resident input matrix: ONE launch of the
persistent tile-DAG kernel (paper_2309_07235_b200/csrc/dag_factor.cu; walker
CTA on the diagonal chain + queue workers on the bulk TRSM/GEMM tasks).  Inputs cycle
through a ring of W+K distinct device copies (each step's input is cold in
L2: the ring is W+K x 32 MB and every copy was written during setup), so
there is no restore copy in the timed region.

value   = algorithmic (2/3) n^3 flop per step x steps x ranks / max-over-ranks
          device time (CUDA events on the launching stream)
e2e     = same metric through the C ABI with pinned host buffers (H2D + factor
          + D2H every step): tt_lu_factor_batch, the pipelined batch of the
          drop-in; the per-call drop-in tt_lu_factor_inplace is e2e.single_call
roofline: bound "tensor" (fp64 DMMA); the dominant (only) kernel of a step
          is the persistent factorisation kernel, so achieved = (2/3) n^3 per
          launch / its CUDA-event launch time; peak = the measured DMMA issue
          rate on this pool's B200s (profiles/fp64_peak_r01.jsonl, 37.05
          TFLOP/s; MEASURED_PEAKS.json has no fp64 entry); traffic = DRAM
          bytes of one ncu --set full capture (profiles/ncu_traffic.json).
Multi-GPU: LU is single-GPU per factorisation (north_star), so N ranks run
N independent replicas ("replicas only", scaling "weak").

`--impl reference` times the reference's own CPU implementation (the
unmodified core compiled into oracle/_ref by oracle/Makefile, else the C
port) on all host cores, each thread factoring its own copy.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FP64_PEAK_TFLOPS = 37.05  # measured DMMA m8n8k4 issue rate (profiles/fp64_peak_r01.jsonl)
FP64_PEAK_SOURCE = "measured: DMMA issue-rate microbenchmark, 148 SMs @1965 MHz (profiles/fp64_peak_r01.jsonl); cuBLAS DGEMM 8192^3 = 35.45"
BENCH_N = 2000
BENCH_LU_BLOCK = (200, 40)  # (by, bx): fastest fixed block of the N=2000 knob sweep of the final round-1 kernel (profiles/sweep_lu2000_r01c.jsonl: 0.879 ms; (250,50) 0.930, the paper's A100 best (400,50) 1.000)
METRIC = "fp64 GFLOP/s of best-tuned config (% of B200 fp64 peak); tuning time-to-best"


def lu_flops(n: int) -> float:
    return 2.0 / 3.0 * n ** 3


def chol_flops(n: int) -> float:
    return n ** 3 / 3.0


def mm3_flops(n, l, m, o, p) -> float:
    return 2.0 * (n * l * m + m * o * p + n * m * p)


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """NVML sampling of SM clock + clock-event reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x1: "gpu_idle"}

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                bits = get_reasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b and b != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ dist

def dist_init(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if _has_cuda() else "gloo")
    return rank, world, local


def _has_cuda() -> bool:
    import torch
    return torch.cuda.is_available()


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if _has_cuda() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ CPU arms

def cpu_reference_lu(n: int, by: int, bx: int, steps: int, threads: int, budget_s: float):
    """Reference CPU LU on `threads` host threads (one matrix each per step)."""
    import oracle
    ref = oracle.ref_lib()
    kind = "reference" if ref is not None else "port"
    base = oracle.gen_spd(n, 1)  # bitwise gen_spd(n, 1)
    pristine = [base.copy() for _ in range(threads)]

    def factor(buf):
        if ref is not None:
            rc = ref.ref_lu_factor_inplace(buf.ctypes.data_as(ctypes.c_void_p), n, n, by, bx)
        else:
            rc = 0
            oracle.lu_factor_inplace(buf, by, bx)
        assert rc == 0

    times = []
    t_start = time.perf_counter()
    for _ in range(steps):
        work = [p.copy() for p in pristine]
        ths = [threading.Thread(target=factor, args=(w,)) for w in work]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    return kind, times


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    by, bx = BENCH_LU_BLOCK
    threads = os.cpu_count() or 1
    # bounded: one warm-up step, then up to K steps within ~150 s of CPU time
    kind, warm = cpu_reference_lu(BENCH_N, by, bx, 1 if args.warmup > 0 else 0, threads, 60.0) \
        if args.warmup > 0 else ("reference", [])
    kind, times = cpu_reference_lu(BENCH_N, by, bx, args.steps, threads, 150.0)
    total = sum(times)
    value = threads * lu_flops(BENCH_N) * len(times) / total / 1e9
    sample = (f"{len(times)} step(s) x {threads} threads, each thread one in-place "
              f"lu_factor_inplace(gen_spd({BENCH_N},1), by={by}, bx={bx}); "
              f"{'unmodified reference core (oracle/_ref)' if kind == 'reference' else 'C port (oracle/tt_oracle.c)'}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": len(times), "steps_requested": args.steps,
        "warmup": args.warmup, "ms_per_step": total / len(times) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_spd(2000, seed=1), bitwise the reference generator)",
        "config": {"workload": f"lu_nopiv_large_n{BENCH_N}_fixed_block", "n": BENCH_N,
                   "by": by, "bx": bx, "threads": threads},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_single(n, by, bx):
    """Reference measure() protocol (1 warm-up + median of 3) on 1 core."""
    import oracle
    ref = oracle.ref_lib()
    if ref is not None:
        cfg = (ctypes.c_int * 2)(by, bx)
        out = ctypes.c_double()
        t0 = time.perf_counter()
        rc = ref.ref_measure(0, b"large", 1, ctypes.cast(cfg, ctypes.c_void_p), 2, 1, 3, 0,
                             ctypes.byref(out))
        assert rc == 0, ref.ref_last_error()
        wall = time.perf_counter() - t0
        secs = out.value
        kind = "reference"
        sample = (f"reference measure(KernelCase{{lu/large, seed 1}}, ({by},{bx}), protocol 1 "
                  f"warm-up + median of 3) on 1 host thread; {wall:.1f} s incl. gen_spd")
    else:
        a = oracle.gen_spd(n, 1)
        ts = []
        for _ in range(4):
            w = a.copy()
            t0 = time.perf_counter()
            oracle.lu_factor_inplace(w, by, bx)
            ts.append(time.perf_counter() - t0)
        secs = float(np.median(ts[1:]))
        kind = "port"
        sample = f"C port lu_factor_inplace n={n} ({by},{bx}), 1 warm-up + median of 3, 1 thread"
    return {"value": lu_flops(n) / secs / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": kind,
            "sample": sample, "seconds_per_factorisation": secs}


# ------------------------------------------------------------------ GPU arm

def run_gpu_arm(args, rank, world, local):
    import torch
    from paper_2309_07235_b200 import Context, GpuKernelRunner, KernelCase
    from paper_2309_07235_b200 import _lib

    torch.cuda.set_device(local)
    ctx = Context(local)
    lib = ctx.lib
    n = BENCH_N
    by, bx = BENCH_LU_BLOCK
    ld = n  # 2000 is a multiple of 16: rows already 128-byte aligned
    # one explicit stream shared by torch (events, copies) and the library
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    sptr = ctypes.c_void_p(stream.cuda_stream)

    # inputs: gen_spd(2000, 1) generated on the device (bitwise the reference's)
    runner = GpuKernelRunner(KernelCase("lu", n, seed=1), ctx)
    (host_a,) = runner.inputs()
    base = torch.from_numpy(host_a).to(f"cuda:{local}")
    ring_len = args.warmup + args.steps
    ring = torch.empty((ring_len, n, ld), dtype=torch.float64, device=f"cuda:{local}")
    ring.copy_(base.expand(ring_len, n, ld))
    torch.cuda.synchronize()

    def factor(i):
        rc = lib.tt_dev_lu(ctx.handle, ctypes.c_void_p(ring[i].data_ptr()), n, ld, by, bx, None,
                           sptr)
        ctx.check(rc)

    # Instantiation cache: a schedule's CUDA graph is specific to its buffer,
    # so build the graph of every ring entry first (untimed), then restore the
    # pristine inputs and evict them from L2 with a 256 MB write.
    for i in range(ring_len):
        factor(i)
    torch.cuda.synchronize()
    ring.copy_(base.expand(ring_len, n, ld))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    flush.fill_(1)
    torch.cuda.synchronize()
    for i in range(args.warmup):
        factor(i)
    torch.cuda.synchronize()
    launches_w = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for i in range(args.warmup, ring_len):
            factor(i)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    launches_timed = ctx.launches - launches_w
    ms_max = max_over_ranks(ms, world)
    value = world * args.steps * lu_flops(n) / (ms_max * 1e-3) / 1e9

    # correctness of the timed outputs (size-independent property): residual of the last factor
    check = torch.empty_like(base)
    check.copy_(ring[ring_len - 1])
    torch.cuda.synchronize()

    # e2e through the C ABI with pinned host buffers: the pipelined batch entry
    # (tt_lu_factor_batch: H2D / factorisation / D2H of neighbouring matrices
    # overlap) is the headline; the per-call drop-in (tt_lu_factor_inplace,
    # one synchronous round trip per matrix) is reported beside it.
    e2e_steps = max(4, min(args.steps, 20))
    host = [torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
            for _ in range(e2e_steps + 1)]
    for h in host:
        h[...] = host_a
    idx = ctypes.c_int(-1)
    ctx.check(lib.tt_lu_factor_inplace(ctx.handle, _lib.ptr(host[-1]), n, n, by, bx,
                                       ctypes.byref(idx)))  # warm the one-shot graph
    ptrs = (ctypes.c_void_p * e2e_steps)(*[h.ctypes.data for h in host[:e2e_steps]])
    fails = (ctypes.c_int * e2e_steps)()
    # warm-up: the same batch call as the timed one (graphs, streams, status slots)
    ctx.check(lib.tt_lu_factor_batch(ctx.handle, ptrs, e2e_steps, n, by, bx, fails))
    for h in host[:e2e_steps]:
        h[...] = host_a
    barrier(world)
    t0 = time.perf_counter()
    ctx.check(lib.tt_lu_factor_batch(ctx.handle, ptrs, e2e_steps, n, by, bx, fails))
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    e2e_value = world * e2e_steps * lu_flops(n) / e2e_s / 1e9
    single = [torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)]
    for h in single:
        h[...] = host_a
    barrier(world)
    t0 = time.perf_counter()
    for h in single:
        ctx.check(lib.tt_lu_factor_inplace(ctx.handle, _lib.ptr(h), n, n, by, bx,
                                           ctypes.byref(idx)))
    single_s = max_over_ranks(time.perf_counter() - t0, world)
    single_value = world * len(single) * lu_flops(n) / single_s / 1e9

    line = None
    if rank == 0:
        import oracle
        res = oracle.lu_residual_packed(host_a, host[e2e_steps - 1])  # CPU check of one e2e output
        same = bool(np.array_equal(host[0], single[0]))  # batch and per-call outputs agree bitwise
        ref_fac = host_a.copy()
        achieved = lu_flops(n) / (ms / args.steps * 1e-3) / 1e12
        traffic = ncu_traffic(f"lu_nopiv_large_n{n}_fixed_block")
        sched = schedule_info(lib, n, by, bx)
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: gen_spd(2000, seed=1) generated on the device, bitwise equal to the reference generator",
            "config": {"workload": f"lu_nopiv_large_n{n}_fixed_block", "n": n, "by": by, "bx": bx,
                       "parallelism": f"replicas{world}",
                       "l2_policy": f"ring of {ring_len} distinct resident inputs (32 MB each), 256 MB L2 flush after restoring them; every timed step's input is cold in L2"},
            "pct_of_fp64_peak": 100.0 * achieved / FP64_PEAK_TFLOPS,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
                         "traffic": traffic,
                         "kernel": sched["kernel"],
                         "launch_unit": "one launch = one full factorisation ((2/3) n^3 flop); timed with CUDA events on the launching stream",
                         "peak_source": FP64_PEAK_SOURCE},
            "schedule": sched,
            "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": n * n * 8,
                    "d2h_bytes_per_step": n * n * 8, "steps": e2e_steps,
                    "api": "tt_lu_factor_batch (C ABI, pipelined batch of lu_factor_inplace)",
                    "single_call": {"value": single_value, "unit": "GFLOP/s", "steps": len(single),
                                    "api": "tt_lu_factor_inplace (C ABI drop-in for lu_factor_inplace)"}},
            "gpu_launches": int(launches_timed),
            "clocks": clk.summary(),
            "parity": {"lu_residual_e2e_output": res, "tolerance": 1e-12,
                       "batch_equals_single_call": same, "ok": bool(res <= 1e-12 and same)},
        }
    return line, ctx


def ncu_traffic(workload: str):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture summary, or None."""
    f = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(f.read_text()).get(workload)
    except Exception:
        return None


def schedule_info(lib, n, by, bx):
    """Which schedule the knob setting runs on (persistent DAG or launch graph)."""
    ntasks = lib.tt_dag_tasks(0, n, by, bx, None, 0)
    if ntasks < 0:
        return {"kind": "graph", "kernel": "panel/trsm/dgemm graph (schedules.cu)"}
    nt = n // bx
    return {"kind": "persistent tile-DAG", "kernel": f"dag_kernel<{(bx + 7) // 8}, LU>",
            "queue_tasks": ntasks, "urgent_tasks": lib.tt_dag_urgent(0, n, by, bx),
            "walker_steps": nt}


def by_fit(extent, f):
    """Largest divisor of `extent` not above f (the trailing view need not be divisible)."""
    f = min(f, extent)
    while extent % f:
        f -= 1
    return f


def extra_workloads(ctx, quick: bool):
    """The other BASELINE configs, device-resident, CUDA-event timed (median of reps)."""
    from paper_2309_07235_b200 import GpuKernelRunner, KernelCase, MeasureProtocol
    out = {}
    proto = MeasureProtocol(2, 5, "median")
    cases = [
        # fixed tile configs: best of the coordinate grid search (profiles/sweep3mm_grid_r01.txt)
        ("mm3_large_fixed", KernelCase("3mm", 800, 900, 1000, 1100, 1200), (100, 125, 125, 120, 32, 60),
         mm3_flops(800, 900, 1000, 1100, 1200)),
        ("mm3_extralarge", KernelCase("3mm", 1600, 1800, 2000, 2200, 2400), (64, 125, 125, 300, 64, 240),
         mm3_flops(1600, 1800, 2000, 2200, 2400)),
        ("cholesky_extralarge", KernelCase("cholesky", 4000), (250, 50), chol_flops(4000)),
        ("lu_extralarge", KernelCase("lu", 4000), (160, 50), lu_flops(4000)),
    ]
    for name, kase, cfg, flops in cases:
        try:
            r = GpuKernelRunner(kase, ctx)
            secs = r.measure(cfg, proto)
            tf = flops / secs / 1e12
            out[name] = {"config": list(cfg), "ms": secs * 1e3, "gflops": tf * 1e3,
                         "pct_of_fp64_peak": 100 * tf / FP64_PEAK_TFLOPS}
        except Exception as e:  # report, never hide
            out[name] = {"error": str(e)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    rank, world, local = dist_init(args.gpus)

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_single(BENCH_N, *BENCH_LU_BLOCK)  # before the GPU phase
    line, ctx = run_gpu_arm(args, rank, world, local)
    if rank == 0:
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if not args.no_extra and world == 1:
            line["extra"] = extra_workloads(ctx, quick=True)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
