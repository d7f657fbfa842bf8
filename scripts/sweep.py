#!/usr/bin/env python3
"""Config 5 sweep (BASELINE.json configs[4]): MARS(15,15), 2 robots, 256
depth-1 leaves, K = 500 ... 32768, on this box's GPUs (one bench.py run per
K; with --gpus N > 1 each run goes through torchrun and the scenario-sharded
NCCL path).  Prints one JSON line per K (bench.py's line)."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--K", type=int, nargs="*", default=[500, 1024, 2048, 4096, 8192, 16384, 32768])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    for K in args.K:
        steps = args.steps if K <= 8192 else max(3, args.steps // 2)
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "5", "--K", str(K), "--steps", str(steps),
               "--warmup", "3", "--no-cpu-baseline", "--gpus", str(args.gpus)]
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr", "127.0.0.1", "--master-port", "29533"] + cmd[1:]
        out = subprocess.run(cmd, capture_output=True, text=True)
        line = [x for x in out.stdout.splitlines() if x.startswith("{")]
        if not line:
            print(json.dumps({"K": K, "error": out.stderr[-500:]}), flush=True)
            continue
        d = json.loads(line[0])
        print(json.dumps({"K": K, "gpus": args.gpus, "value": d["value"], "ms_per_step": d["ms_per_step"],
                          "frac": d["roofline"]["frac"], "k2_ms": d["phases_ms"]["K2_expand_rollout"],
                          "steps_per_batch": d["config"]["scenario_steps_per_batch"]}), flush=True)


if __name__ == "__main__":
    main()
