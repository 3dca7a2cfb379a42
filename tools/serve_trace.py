"""BASELINE.json configs[3]: ViT-B/16 selective-batching serving trace, mixed-SLO synthetic
query stream, replicas on N B200s.

  python tools/serve_trace.py [--gpus N] [--duration S] [--rate-scale K] [--out DIR]

1. builds one ServeModel replica per GPU (CIFAR10 / CIFAR100 / EuroSAT heads, prompts for the
   gamma list's positive values; random-init weights);
2. profiles replica 0 on the device (per-sample latency per (task, gamma) at batch 64 = the
   batcher's epsilon) -> ProfileTable (written as the kind,task,gamma,batch_size,value CSV);
   accuracy comes from engine.synthetic_accuracy (random weights: no real accuracy);
3. derives f (rate -> gamma) from the measured throughput of N replicas;
4. generates the paper's synthetic workload (Poisson, query types of PAPER.md:579-595, rate
   drawn per second in [200, 700] req/s) scaled by --rate-scale to load B200s;
5. serves it with OTAS (Alg. 1-3) and the fixed-gamma baselines (ToMe -20, PetS 0, VPT +8),
   every planned batch executing on a GPU replica; prints one JSON line per policy and writes
   the metric CSVs (utility curve, accuracy CDF, gamma ratio, outcome ratio) under --out.
"""
import argparse
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2401_05031_b200.adapter import PAPER_GAMMAS, AdapterConfig  # noqa: E402
from paper_2401_05031_b200.engine import (DEFAULT_TASKS, AsyncGpuExecutor, EngineConfig, GpuExecutor,  # noqa: E402
                                          ServingEngine, build_replicas, synthetic_accuracy)
from paper_2401_05031_b200.profiles import RateToGammaMap, derive_f, write_profile_csv  # noqa: E402
from paper_2401_05031_b200.workload import gen_poisson  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=torch.cuda.device_count())
    ap.add_argument("--model", default="vit_b16")
    ap.add_argument("--duration", type=float, default=6.0)
    ap.add_argument("--rate-scale", type=float, default=40.0)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--policies", default="otas,-20,0,8")
    ap.add_argument("--out", default="gpurun_out/serve_trace")
    ap.add_argument("--dp-horizon", type=int, default=16, help="Alg. 2 over the earliest-deadline K batches per plan")
    ap.add_argument("--frontier-cap", type=int, default=16, help="DP frontier states per row")
    ap.add_argument("--clock", default="realtime", choices=["realtime", "virtual"],
                    help="realtime: replicas execute concurrently against the wall clock (AsyncGpuExecutor); "
                         "virtual: deterministic discrete-event clock, batches executed one at a time")
    args = ap.parse_args()
    gammas = PAPER_GAMMAS
    devices = [f"cuda:{i}" for i in range(args.gpus)]
    replicas, index = build_replicas(args.model, devices, DEFAULT_TASKS, gammas.values)
    t0 = time.time()
    table = replicas[0].profile(gammas.values, 64, synthetic_accuracy(DEFAULT_TASKS, gammas.values), iters=3, warmup=2)
    os.makedirs(args.out, exist_ok=True)
    write_profile_csv(table, os.path.join(args.out, "profile_b200.csv"))
    f1 = derive_f(table, gammas, 64)
    f = RateToGammaMap(tuple((lo * args.gpus if i else lo, g) for i, (lo, g) in enumerate(f1.breakpoints)))
    adapter = AdapterConfig(gammas=gammas, rate_map=f)
    rng = random.Random(args.seed)
    profile = [(s, rng.uniform(200, 700) * args.rate_scale) for s in range(int(args.duration))]
    if args.clock == "realtime":
        executor = AsyncGpuExecutor([r.backbone for r in replicas], index)
    else:
        executor = GpuExecutor([r.backbone for r in replicas], index)
    results = {}
    for pol in args.policies.split(","):
        policy = pol if pol == "otas" else int(pol)
        qs = gen_poisson(profile, args.duration, seed=args.seed)
        w0 = time.time()
        ecfg = EngineConfig(policy=policy, seed=args.seed, dp_horizon=args.dp_horizon, frontier_cap=args.frontier_cap)
        eng = ServingEngine(executor, table, adapter=adapter, cfg=ecfg)
        rep = eng.run_realtime(qs) if args.clock == "realtime" else eng.run(qs)
        wall = time.time() - w0
        rep.export(os.path.join(args.out, f"policy_{pol}"))
        s = rep.summary()
        line = {"config": "ViT-B/16 selective-batching serving trace (configs[3])", "policy": pol,
                "gpus": args.gpus, "rate_scale": args.rate_scale, "duration_s": args.duration,
                "offered_rps": round(len(qs) / args.duration, 1), "utility": s["utility"],
                "served_ratio": s["served_ratio"], "outcomes": s["outcomes"], "gamma_counts": s["gamma_counts"],
                "executed_images": s["executed_images"],
                "served_images_per_s_virtual": round(s["executed_images"] / max(s["end_s"], 1e-9), 1),
                "gpu_busy_frac": [round(b / max(s["end_s"], 1e-9), 3) for b in s["busy_s"]],
                "host_wall_s": round(wall, 2), "clock": args.clock, "dp_horizon": args.dp_horizon,
                "frontier_cap": args.frontier_cap}
        results[pol] = line
        print(json.dumps(line), flush=True)
    print(json.dumps({"rate_map": f.breakpoints, "profile_s": round(time.time() - t0, 1)}), flush=True)
    if hasattr(executor, "close"):
        executor.close()


if __name__ == "__main__":
    main()
