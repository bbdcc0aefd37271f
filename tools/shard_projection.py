"""Strong-scaling projection for the C5 walk from ONE GPU: every shard of an
N-way split (the exact [k_begin, k_end) ranges perm_walk_shard hands to
ranks 0..N-1) is timed on this device with CUDA events, and the projected
N-GPU time is max over shards (the all-gather of 8 doubles per rank is not
included; NCCL over NVLink takes tens of microseconds for it).  This is the
compute-side bound on scaling efficiency T1 / (N * T_N), measured; the real
multi-GPU number comes from `bench.py --gpus N` under torchrun.

    python tools/shard_projection.py [n=36] > gpurun_out/shard_projection.json
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    from paper_2510_03421_b200 import workloads as W
    from paper_2510_03421_b200.sharded import gpu_partial, shard_range

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 36
    a = W.c5(n)
    stream = torch.cuda.current_stream()
    part = torch.zeros(8, dtype=torch.float64, device="cuda")

    def timed(k0, k1, reps):
        gpu_partial("glynn", a, k0, k1, False, device_out=part, stream=stream.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            gpu_partial("glynn", a, k0, k1, False, device_out=part, stream=stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    t1 = timed(*shard_range("glynn", n, n, 0, 1), 3)
    out = {"n": n, "t1_ms": t1, "projection": {}}
    for N in (2, 4, 8):
        ts = [timed(*shard_range("glynn", n, n, r, N), 3) for r in range(N)]
        out["projection"][str(N)] = {"shard_ms": ts, "t_ms": max(ts), "efficiency": t1 / (N * max(ts))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
