"""Benchmark driver (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c1|c4|c5]

Workloads (BASELINE.json configs):
  c2 (default): full Mistral-7B-shaped decoder stack, 3 experts with 2-bit + fp16-salient
      deltas on all 224 decoder linears, mixed-expert batch decode (one step = one token
      for every request in the batch).
  c1: one 4096x14336 MLP linear, 3 experts, batch-8 mixed decode (the CPU-runnable case).
  c4: prefill of 2048 tokens over 16 experts through the same linear (tensor-bound roofline).
  c5: 64 experts sharded over the N GPUs (64/N per GPU, expert e on rank e mod N), batch 128
      per GPU through the c2 decode engine (with --gpus 1 all 64 experts are resident on one GPU).

The default c2 line (N=1) also carries, measured in the same process outside the timed
region: `c1` (the C1 kernel line), `c3` (16 router-assigned experts, B=128), `parity`
(sampled layer vs the f64 restatement), `delta_gemm` (delta-only launches), `router`.

--gpus N without WORLD_SIZE re-launches itself under torchrun (one process per GPU).

Under torchrun (N>1) every rank serves its own expert shard (experts placed e mod G,
replicated base, no collective on the data path): weak scaling, value = all tokens / max time.
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

import numpy as np  # noqa: E402


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c4", "c5"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--experts", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="c2 only: skip the same-process C1/C3/parity legs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (the driver does the same)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MESW_MASTER_PORT", "29517"),
               os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if ws != args.gpus:
        print(f"[bench] warning: --gpus {args.gpus} but WORLD_SIZE={ws}; using {ws} rank(s)", file=sys.stderr)

    if args.impl == "reference":
        from bench_impl import reference_arm
        if rank != 0:
            return 0
        try:  # torchrun sets OMP_NUM_THREADS=1 per rank; the reference arm is rank 0 alone: use all cores
            from threadpoolctl import threadpool_limits
            threadpool_limits(os.cpu_count())
        except Exception:
            pass
        line = reference_arm(args)
        print(json.dumps(line), flush=True)
        return 0

    import torch
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"[bench] rank {rank}/{ws} on cuda:{local} ({torch.cuda.get_device_name(local)}), "
              f"process group size {dist.get_world_size()}", file=sys.stderr, flush=True)
    from bench_impl import run_ours
    line = run_ours(args, ws, rank, local, ClockSampler, _peaks)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
