#!/usr/bin/env python
"""Benchmark driver (one JSON line on rank 0).

Headline workload: BASELINE.json configs[4] = C5, the large single float64
permanent n = 36 (entries iid U[0,1]/36, seeded), computed with the Gray-code
Glynn walk; its 2^35 sign vectors are sharded over the N ranks (one GPU
each, NCCL all-gather of 8-double partials), so the total work is fixed as N
grows ("strong" scaling).  metric = Gray-code steps/s of the whole job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 36]
    python bench.py --impl reference ...   # the reference's CPU algorithm
                                           # (oracle C port, all host threads)

A "step" is one full permanent.  Timing: barrier + cuda.synchronize around
the timed region, CUDA events on the launching stream per step (L2 flushed
with a 256 MiB write before every step, outside the events), max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Gray-code steps/sec and s/permanent at n=20–36; % of FP64 FMA peak, 1/2/4/8 GPUs"
UNIT = "steps/s"
NOMINAL_DFMA = 148 * 64 * 1965e6  # FP64 pipe slots/s at the max SM clock


def workload_name(n):
    return f"C5: Glynn f64 {n}x{n} U[0,1]/{n} single permanent, 2^{n - 1} Gray steps sharded over ranks"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------- CPU baseline
def cpu_walk_rate(a: np.ndarray, nthreads: int, target_s: float):
    """Oracle port (perm_oracle.c, the reference's sequential Glynn walk
    restated in C) over a bounded prefix of the same walk: steps/s."""
    from oracle import oracle as O

    setup = O.walk_setup("glynn", a)
    steps = 1 << 22
    t = time.perf_counter()
    O.walk_f64_mt(setup, 0, steps, nthreads=nthreads)
    dt = time.perf_counter() - t
    steps = int(min(1 << (a.shape[1] - 1), max(steps, steps * target_s / max(dt, 1e-6))))
    steps -= steps % nthreads
    t = time.perf_counter()
    O.walk_f64_mt(setup, 0, steps, nthreads=nthreads)
    dt = time.perf_counter() - t
    return steps / dt, steps, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2510_03421_b200 import workloads as W

    O.build()
    a = W.c5(args.n)
    cores = os.cpu_count() or 1
    # calibrate a per-step sample of ~target seconds
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    rate, sample, _ = cpu_walk_rate(a, cores, per_step)
    for _ in range(args.warmup):
        cpu_walk_rate_fixed(O, a, sample, cores)
    times = [cpu_walk_rate_fixed(O, a, sample, cores) for _ in range(args.steps)]
    total = sum(times)
    value = sample * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded U[0,1]/n, SURVEY 8(d) k=8)",
        "config": {"workload": workload_name(args.n), "n": args.n,
                   "sample_steps_per_step": sample, "s_per_permanent_extrapolated":
                   (1 << (args.n - 1)) / value},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"first {sample} Gray steps of the {args.n}x{args.n} C5 walk per step, "
                                   f"split over {cores} threads (oracle/perm_oracle.c, the reference's "
                                   "src/_kernels.py:373-409 walk restated; reference itself is Python+numba, "
                                   "not present on the GPU box)",
                         "port_vs_reference": "the port's 1-thread rate on this box (bench.py cpu_baseline, "
                                              "3.0-4.3e7 steps/s) matches the numba reference's single-threaded "
                                              "glynn_sq measured in the build container (2.7-5.2e7 steps/s, "
                                              "SURVEY 6); the reference walk is single-threaded, so this "
                                              "all-threads port is a stronger CPU baseline than the reference"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def cpu_walk_rate_fixed(O, a, steps, nthreads):
    setup = O.walk_setup("glynn", a)
    t = time.perf_counter()
    O.walk_f64_mt(setup, 0, steps, nthreads=nthreads)
    return time.perf_counter() - t


def check_value(n: int, v: float) -> dict:
    """Self-check of the benchmarked result against the committed GPU
    double-double Ryser value (tests/golden/c5_dd.json): fail loudly when
    the relative error exceeds 1e-10, or the scale-aware metric (ii) does."""
    ref = json.loads((ROOT / "tests" / "golden" / "c5_dd.json").read_text())
    dd = ref["ryser_dd"].get(str(n))
    if dd is None:
        return {"value": v, "checked": False}
    rel = abs(v - dd) / max(abs(v), abs(dd))
    M = ref["glynn_magsum"].get(str(n), abs(dd))
    scaled = abs(v - dd) / max(abs(v), abs(dd), M)
    if rel > 1e-10 or scaled > 1e-10:
        raise SystemExit(f"bench: C5 n={n} value {v!r} differs from the double-double Ryser {dd!r} "
                         f"(rel {rel:.3e}, scaled {scaled:.3e})")
    return {"value": v, "checked": True, "ref_ryser_dd": dd, "rel_err": rel, "scaled_err": scaled}


def measure_configs(P, W, torch) -> dict:
    """BASELINE configs[0..3] on one GPU: median wall clock of the public
    call on host numpy input, device time for device-resident batches."""
    def wall(fn, reps=5, warm=2):
        for _ in range(warm):
            fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts)

    out = {}
    c1 = W.c1()
    out["C1_glynn_batch_64x12x12"] = {"e2e_ms": 1e3 * wall(lambda: P.glynn_batch(c1), reps=11)}
    for name, A in (("C2a_opt_batch_1e6x8x8", W.c2a()), ("C2b_opt_batch_1e6x4x10", W.c2b())):
        e2e = wall(lambda: P.opt_batch(A), reps=3, warm=1)
        pA = torch.from_numpy(A).pin_memory()  # page-locked input: the DMA reads it in place
        e2e_pinned = wall(lambda: P.opt_batch(pA), reps=3, warm=1)
        del pA
        dA = torch.tensor(A, device="cuda")
        P.opt_batch(dA)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            P.opt_batch(dA)
        e1.record()
        torch.cuda.synchronize()
        dev_ms = e0.elapsed_time(e1) / 10
        out[name] = {"e2e_ms": 1e3 * e2e, "e2e_pinned_ms": 1e3 * e2e_pinned,
                     "h2d_gbs_pinned": A.nbytes / e2e_pinned / 1e9, "device_ms": dev_ms,
                     "hbm_gbs_device": A.nbytes / (dev_ms * 1e-3) / 1e9}
        del dA
    c3 = json.loads((ROOT / "tests" / "golden" / "c3.json").read_text())
    for name, a, key in (("C3a_glynn_c128_24x24", W.c3a(), "c3a"), ("C3b_glynn_c128_20x28", W.c3b(), "c3b")):
        v = P.glynn(a)
        ref = complex(c3[f"{key}_dd_glynn"]["re"], c3[f"{key}_dd_glynn"]["im"])
        out[name] = {"e2e_ms": 1e3 * wall(lambda: P.glynn(a)),
                     "rel_err_vs_dd": abs(v - ref) / max(abs(v), abs(ref))}
    c4 = json.loads((ROOT / "tests" / "golden" / "c4.json").read_text())
    for name, a, key in (("C4a_glynn_int128_01_n32", W.c4a(), "c4a"), ("C4b_glynn_int128_pm2_n28", W.c4b(), "c4b")):
        v = P.glynn(a, exact="int128")
        t = wall(lambda: P.glynn(a, exact="int128"), reps=3, warm=1)
        # which exact walk ran (report the pipe): the est_kind
        # slot of the width-128 partial, 3 / 4 = the quad walk (packed FP32
        # state, FP64 pair products, integer last level), 1 = FP64-exact groups
        from paper_2510_03421_b200 import sharded as S
        kind = int(S.gpu_partial_int("glynn", a, 0, 1 << (a.shape[1] - 1), exact="int128")[5])
        out[name] = {"e2e_ms": 1e3 * t, "steps_per_s": (1 << (a.shape[1] - 1)) / t,
                     "walk": {4: "quad walk: FP32x2 + FP64 + IMAD pipes", 3: "quad walk: FP32x2 + IMAD pipes",
                              1: "FP64-exact groups + IMAD"}.get(kind, f"est_kind {kind}"),
                     "exact_matches_fixture": str(v) == str(c4[f"{key}_exact"])}
    return out


# ------------------------------------------------------------- engine arm
def run_engine(args):
    # stdout carries the JSON line only: under torchrun, NCCL prints its
    # version banner to the process's stdout (NCCL_DEBUG=VERSION is set in
    # the GPU image), so file descriptor 1 points at stderr for the run and
    # the JSON line is written to the saved descriptor
    json_fd = None
    if "WORLD_SIZE" in os.environ:
        sys.stdout.flush()
        json_fd = os.dup(1)
        os.dup2(2, 1)
    try:
        return _run_engine(args, json_fd)
    finally:
        if json_fd is not None:
            sys.stdout.flush()
            os.dup2(json_fd, 1)
            os.close(json_fd)


def _emit(line: dict, json_fd):
    text = json.dumps(line)
    if json_fd is None:
        print(text, flush=True)
    else:
        os.write(json_fd, (text + "\n").encode())


def _run_engine(args, json_fd):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # under torchrun (WORLD_SIZE set) the NCCL path runs even for N = 1
    distributed = "WORLD_SIZE" in os.environ
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2510_03421_b200 as P
    from paper_2510_03421_b200 import _lib, workloads as W
    from paper_2510_03421_b200.sharded import finish, gpu_partial, shard_range

    lib = _lib.load()
    _lib.check(lib.perm_set_device(local), "set_device")
    lib.perm_set_timing(1)  # CUDA events around each walk kernel (roofline)
    n = args.n
    a = W.c5(n)
    k0, k1 = shard_range("glynn", n, n, rank, world)
    steps_total = 1 << (n - 1)
    stream = torch.cuda.current_stream()
    part = torch.zeros(8, dtype=torch.float64, device="cuda")
    gathered = torch.zeros(8 * world, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step():
        gpu_partial("glynn", a, k0, k1, False, device_out=part, stream=stream.cuda_stream)
        if distributed:
            dist.all_gather_into_tensor(gathered, part)
        else:
            gathered.copy_(part)

    # FP64-pipe roofline denominators, measured live on this GPU: DFMA chains
    # (the metric's "FMA peak") and DADD/DMUL chains (the walk's own mix,
    # which reaches the nominal rate); the roofline uses the larger
    peak = _lib.out_buf(1)
    _lib.check(lib.perm_fp64_pipe_probe(0, 1.0, peak), "peak probe")
    peak_dfma = float(peak[0])
    _lib.check(lib.perm_fp64_pipe_probe(1, 1.0, peak), "peak probe")
    peak_addmul = float(peak[0])
    peak_pipe = max(peak_dfma, peak_addmul)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    value_check, _ = finish("glynn", a, gathered.cpu().numpy())
    check = check_value(n, value_check)

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    kernel_ms = []
    for i in range(args.steps):
        flush.fill_(float(i))  # > 126 MB L2, outside the timed events
        ev[i][0].record(stream)
        gpu_partial("glynn", a, k0, k1, False, device_out=part, stream=stream.cuda_stream)
        ev[i][1].record(stream)  # walk done: [1] -> [2] is the exchange
        if distributed:
            dist.all_gather_into_tensor(gathered, part)
        else:
            gathered.copy_(part)
        ev[i][2].record(stream)
        kernel_ms.append(lib.perm_last_kernel_ms())
    torch.cuda.synchronize()
    # per-rank breakdown (walk kernel, walk call, exchange), gathered to rank 0
    mine = torch.tensor([statistics.mean(kernel_ms), statistics.mean(s.elapsed_time(m) for s, m, _ in ev),
                         statistics.mean(m.elapsed_time(e) for _, m, e in ev), float(k1 - k0)],
                        dtype=torch.float64, device="cuda")
    per_rank = torch.zeros(4 * world, dtype=torch.float64, device="cuda")
    if distributed:
        dist.all_gather_into_tensor(per_rank, mine)
    else:
        per_rank.copy_(mine)
    per_rank = [dict(zip(("walk_kernel_ms", "walk_call_ms", "exchange_ms", "gray_steps"), map(float, r)))
                for r in per_rank.view(world, 4).cpu().tolist()]
    if distributed:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    t_ms = sum(s.elapsed_time(e) for s, _, e in ev)
    t = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    grid, log2L = _lib.C.c_int(), _lib.C.c_int()
    lib.perm_last_kernel_plan(_lib.C.byref(grid), _lib.C.byref(log2L))

    value = steps_total * args.steps / (t_ms * 1e-3)
    kern_ms = statistics.mean(kernel_ms)
    ops_per_launch = (k1 - k0) * 2 * n  # 2n FP64-pipe ops per Glynn step
    achieved = ops_per_launch / (kern_ms * 1e-3)

    # ---- e2e through the public API (host numpy input -> Python float) --
    if distributed:
        dist.barrier()
    e2e_times = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        v = P.sharded_permanent(a) if distributed else P.glynn(a)
        e2e_times.append(time.perf_counter() - t0)
    e2e = torch.tensor([sum(e2e_times)], dtype=torch.float64, device="cuda")
    if distributed:
        dist.all_reduce(e2e, op=dist.ReduceOp.MAX)
    e2e_value = steps_total * args.steps / float(e2e.item())

    # ---- n-sweep (the metric's "n = 20-36"): single-GPU permanents on rank
    # 0, same seeded law (SURVEY 8(d) k = 10 + n).  call_ms: median wall clock
    # of the public call P.glynn / P.ryser on a host numpy matrix (setup,
    # launch, result back in Python -- the per-permanent latency a user
    # sees); device_ms: the walk kernel's device time per permanent,
    # launched back to back with its setup resident (perm_walk_repeat_ms,
    # launch-to-launch gaps included), which frac_of_pipe is computed from
    sweep = {}
    if rank == 0:
        for alg, ns in (("glynn", 20), ("glynn", 22), ("glynn", 24), ("glynn", 26), ("glynn", 28), ("glynn", 30),
                        ("glynn", 32), ("glynn", 34), ("ryser", 24), ("ryser", 28), ("ryser", 32)):
            asw = np.ascontiguousarray(W.c5(ns))
            tot = (1 << (ns - 1)) if alg == "glynn" else (1 << ns)
            fn = P.glynn if alg == "glynn" else P.ryser
            for _ in range(3):
                fn(asw)
            reps = 101 if ns <= 24 else (11 if ns <= 28 else 3)
            walls = []
            for _ in range(reps):
                t0 = time.perf_counter()
                fn(asw)
                walls.append(time.perf_counter() - t0)
            dev = _lib.out_buf(1)
            code = _lib.ALG_GLYNN if alg == "glynn" else _lib.ALG_RYSER
            _lib.check(lib.perm_walk_repeat_ms(code, 0, ns, ns, _lib.C.c_void_p(asw.ctypes.data), ns,
                                               200 if ns <= 24 else (20 if ns <= 28 else 3), dev), "repeat")
            dms = float(dev[0])
            key = str(ns) if alg == "glynn" else f"ryser_{ns}"
            sweep[key] = {"call_ms": 1e3 * statistics.median(walls), "device_ms": dms,
                          ("steps_per_s" if alg == "glynn" else "subsets_per_s"): tot / (dms * 1e-3),
                          "frac_of_pipe": tot * 2 * ns / (dms * 1e-3) / peak_pipe}
            if alg == "glynn" and ns <= 26:
                # throughput of the same size through the batch entry point (B
                # independent matrices of the same law, device resident, one
                # segmented walk launch): what a caller with many n x n
                # permanents gets; a single small permanent is launch-latency bound
                Bn = 1 << (29 - ns)
                rb = np.random.default_rng([2510, 3421, 10 + ns, 1])
                dA = torch.tensor(rb.uniform(0, 1, (Bn, ns, ns)) / ns, device="cuda")
                P.glynn_batch(dA)
                torch.cuda.synchronize()
                b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                b0.record()
                for _ in range(5):
                    P.glynn_batch(dA)
                b1.record()
                torch.cuda.synchronize()
                bms = b0.elapsed_time(b1) / 5
                sweep[key].update({"batch_B": Bn, "batch_ms": bms, "batch_steps_per_s": Bn * tot / (bms * 1e-3),
                                   "batch_frac_of_pipe": Bn * tot * 2 * ns / (bms * 1e-3) / peak_pipe})
                del dA

    # ---- the other BASELINE configs (rank 0, outside the timed region):
    # public-API wall clock on host inputs (e2e) and, for the device-resident
    # batches, the kernel's device time; each checked against its committed
    # reference value where one exists (tests/golden)
    configs = {}
    if rank == 0 and not args.no_configs:
        configs = measure_configs(P, W, torch)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O

        O.build()
        rate, sample, dt = cpu_walk_rate(a, 1, args.cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"first {sample} Gray steps of the same {n}x{n} walk on 1 host thread "
                         f"({dt:.1f} s; oracle/perm_oracle.c restating src/_kernels.py:373-409, which "
                         "is single-threaded in the reference)"}

    traffic = None
    tf = ROOT / "profiles" / "roofline_traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(f"glynn_f64_n{n}")
        except (ValueError, OSError):
            traffic = None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U[0,1]/n matrix, SURVEY 8(d) k=8)",
            "config": {"workload": workload_name(n), "n": n, "alg": "glynn",
                       "s_per_permanent": t_ms * 1e-3 / args.steps,
                       "parallelism": f"gray-range shards x{world} (NCCL all-gather of 8-double partials)",
                       "l2": "flushed (256 MiB write) before every step, outside the timed events",
                       "launch": {"grid": grid.value, "threads": 256, "log2_chunk": log2L.value},
                       "value_check": check,
                       "per_rank": per_rank,
                       "n_sweep_1gpu": sweep,
                       "configs_1gpu": configs},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak_pipe, "unit": "FP64 op/s",
                         "frac": achieved / peak_pipe, "frac_of_fma_peak": achieved / peak_dfma,
                         "frac_of_nominal": achieved / NOMINAL_DFMA,
                         "peak_dfma": peak_dfma, "peak_dadd_dmul": peak_addmul,
                         "traffic": traffic,
                         "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch from the "
                                           "committed ncu --set full capture (profiles/roofline_traffic.json), "
                                           "not measured in this run",
                         "peak_source": "measured live on this GPU, max of two FP64-pipe probes "
                                        "(perm_fp64_pipe_probe: DFMA chains, DADD/DMUL chains); "
                                        "MEASURED_PEAKS.json has no FP64 entry; nominal = 148 SM x 64 "
                                        "op/clk x 1965 MHz",
                         "ops_per_step": 2 * n, "kernel_ms": kern_ms,
                         "kernel_share_of_step": kern_ms / (t_ms / args.steps)},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": (n + (n - 1) * n) * 8,
                    "d2h_bytes_per_step": 8 * 8,
                    "api": "paper_2510_03421_b200.glynn(numpy) / sharded_permanent(numpy) for N>1",
                    "s_per_permanent": float(e2e.item()) / args.steps},
            "gpu_launches": args.steps,  # one walk_kernel per step (block partials combined in-kernel)
            "clocks": clocks,
        }
        _emit(line, json_fd)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=36)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1-C4 section (configs_1gpu)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_engine(args)


if __name__ == "__main__":
    sys.exit(main())
