"""Throughput benchmark of the token-adapted ViT forward on B200 (BASELINE.json metric:
"ViT-B/16 images/sec per gamma (merge/prompt) at 1/2/4/8 B200; roofline fraction").

A step is one sweep over gamma in {-16, -8, 0, +8, +16}: one batch of 256 synthetic
224x224 images per gamma through the full forward (configs[1]).  Each gamma runs as a
CUDA graph of ta_forward.  `value` is images/s over the K timed steps (device time, CUDA
events, L2 flushed before every step, max over ranks), `e2e` is the same metric through
ServeModel.forward with pinned host images (H2D + forward + D2H logits per batch).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: one process per GPU (torchrun), full replica each, no collectives on the path
(replicas only); value = all ranks' images / max-over-ranks time.
--impl reference times the CPU oracle (the reference has no implementation of the path,
SURVEY.md §0; kind "port") on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

GAMMAS = (-16, -8, 0, 8, 16)
METRIC = "ViT-B/16 images/sec per gamma (merge/prompt) at 1/2/4/8 B200; roofline fraction"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained"), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.index, self.samples, self.reasons = index, [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def launches_per_forward(cfg, gamma, prompt_mode="accumulate", fold_ln=True):
    """Kernels one ta_forward launches: patchify, patch GEMM, cls/prompt rows, head; per layer
    [prompt rows], [LN1], QKV, attention, proj, match + merge | [LN2], fc1, fc2 (LN1 / LN2 are
    folded into the QKV / fc1 GEMMs in the default bf16 mode)."""
    from paper_2401_05031_b200.config import token_schedule

    ts, rs = token_schedule(cfg, gamma, prompt_mode)
    n = 3 + 1
    for layer, r in enumerate(rs):
        n += 5 + (0 if fold_ln else 1)
        n += 2 if r > 0 else (0 if fold_ln else 1)
        if gamma > 0 and layer > 0:
            n += 1
    return n


def cpu_oracle_sample(cfg, params, tasks, batch, gammas, seed=0):
    """Times the CPU oracle (fp32, all host threads) over one batch per gamma."""
    from tests import helpers

    n_threads = len(os.sched_getaffinity(0))
    torch.set_num_threads(n_threads)
    imgs = helpers.synthetic_images(batch, cfg.img, seed=seed)
    ids = torch.zeros(batch, dtype=torch.int64)
    t0 = time.perf_counter()
    for g in gammas:
        helpers.oracle_forward(cfg, params, tasks, imgs, ids, g)
    dt = time.perf_counter() - t0
    return batch * len(gammas) / dt, n_threads, dt


def run_reference(args):
    """--impl reference: the CPU oracle (port) on the host cores, bounded sample per step."""
    from paper_2401_05031_b200.config import VIT_CONFIGS
    from tests import helpers

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg, params = helpers.backbone(args.model)
    tasks = helpers.task_params(cfg, (100,), [g for g in GAMMAS if g > 0])
    sample_batch = args.ref_batch
    for _ in range(args.warmup):
        cpu_oracle_sample(cfg, params, tasks, 1, GAMMAS)
    total_imgs, total_t, cores = 0, 0.0, 1
    for s in range(args.steps):
        ips, cores, dt = cpu_oracle_sample(cfg, params, tasks, sample_batch, GAMMAS, seed=s)
        total_imgs += sample_batch * len(GAMMAS)
        total_t += dt
    value = total_imgs / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": f"{args.model} gamma sweep {list(GAMMAS)} (CPU sample: batch {sample_batch} per gamma)",
                   "model": args.model, "global_batch": sample_batch * len(GAMMAS), "seq_len": VIT_CONFIGS[args.model].n_tokens,
                   "parallelism": "cpu", "prompt_mode": "accumulate"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": "port",
                         "sample": f"oracle/vit_oracle.py fp32 torch-CPU, {args.steps} steps x {len(GAMMAS)} gammas x batch {sample_batch}"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch.distributed as dist

    from paper_2401_05031_b200.config import VIT_CONFIGS, flops_per_image
    from tests import helpers

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    # one rank per GPU; if a box exposes fewer GPUs than ranks (multi-rank smoke tests on a
    # single-GPU box) ranks share devices round-robin
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)

    cfg, params = helpers.backbone(args.model)
    gammas = tuple(int(g) for g in args.gammas.split(",")) if args.gammas else GAMMAS
    tasks = helpers.task_params(cfg, (100,), [g for g in gammas if g > 0])
    sm = helpers.serve_model(cfg, params, tasks, dtype="bf16", fold_ln=bool(args.fold_ln))
    bb = sm.backbone
    B = args.batch
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    images = {g: torch.randn(B, 3, cfg.img, cfg.img, generator=gen, device=dev) for g in gammas}
    ids = torch.zeros(B, dtype=torch.int32, device=dev)
    logits = {g: torch.empty(B, bb.max_classes, device=dev) for g in gammas}
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # one CUDA graph per gamma
    graphs = {}
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        for g in gammas:
            for _ in range(2):
                bb.forward_raw(images[g], ids, g, logits=logits[g])
    torch.cuda.current_stream(dev).wait_stream(s)
    torch.cuda.synchronize(dev)
    for g in gammas:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            bb.forward_raw(images[g], ids, g, logits=logits[g])
        graphs[g] = gr
    torch.cuda.synchronize(dev)

    def step(per_gamma_ms=None):
        flush.zero_()  # evict L2 (512 MiB > 126 MB) before every step, outside the events
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(gammas) + 1)]
        evs[0].record()
        for i, g in enumerate(gammas):
            graphs[g].replay()
            evs[i + 1].record()
        return evs

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev_list = []
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.steps):
            ev_list.append(step())
        torch.cuda.synchronize(dev)
    per_gamma_ms = {g: 0.0 for g in gammas}
    total_ms = 0.0
    for evs in ev_list:
        for i, g in enumerate(gammas):
            ms = evs[i].elapsed_time(evs[i + 1])
            per_gamma_ms[g] += ms
            total_ms += ms
    from paper_2401_05031_b200.replicas import aggregate_throughput

    # replicas only: images summed over ranks, device time = max over ranks
    imgs_total, total_ms = aggregate_throughput(args.steps * len(gammas) * B, total_ms)
    if world > 1:
        dist.barrier()
    value = imgs_total / (total_ms / 1e3)
    peak_burst, peak_sus, hbm, peak_src = _peaks()
    # the forward is timed inside a long step (tens of ms of back-to-back tensor work), so the
    # roofline denominator is the SUSTAINED bf16 figure; the burst one is reported beside it
    peak = peak_sus or peak_burst
    flops = {g: flops_per_image(cfg, g) for g in gammas}
    sweep_flops = sum(flops[g] * B for g in gammas) * args.steps
    achieved = sweep_flops / (total_ms / 1e3) / 1e12  # per GPU
    per_gamma = {}
    for g in gammas:
        ips = args.steps * B / (per_gamma_ms[g] / 1e3)
        tf = ips * flops[g] / 1e12
        per_gamma[str(g)] = {"images_per_s": round(ips, 1), "ms_per_batch": round(per_gamma_ms[g] / args.steps, 3),
                             "gflop_per_image": round(flops[g] / 1e9, 3), "tflops": round(tf, 1),
                             "roofline_frac": round(tf / peak, 4), "frac_of_burst": round(tf / peak_burst, 4)}

    # dominant kernel alone: fc1 GEMM at the gamma=0 shape (M = B*197, N = 4D, K = D)
    dom = dominant_gemm(cfg, B, dev, peak_burst)  # timed alone: burst peak

    # e2e through the public API: pinned host images -> ServeModel.forward -> host logits
    e2e_ips, h2d, d2h = run_e2e(sm, cfg, B, gammas, args, dev)
    if world > 1:
        t = torch.tensor([e2e_ips], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)  # slowest replica bounds the job
        e2e_ips = float(t.item()) * world

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        ips, cores, dt = cpu_oracle_sample(cfg, params, tasks, args.cpu_batch, gammas)
        cpu = {"value": round(ips, 3), "unit": "images/s", "cores": cores, "kind": "port",
               "sample": f"oracle/vit_oracle.py fp32 torch-CPU, one batch of {args.cpu_batch} per gamma {list(gammas)} ({dt:.1f} s)"}

    launches = args.steps * sum(launches_per_forward(cfg, g, fold_ln=bool(args.fold_ln)) for g in gammas)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.model} batch {B} per gamma, sweep gamma in {list(gammas)}"
                                   f"{' (configs[1])' if args.model == 'vit_b16' and gammas == GAMMAS and B == 256 else ''}; one step = the sweep",
                       "model": args.model, "global_batch": B * len(gammas) * world, "seq_len": cfg.n_tokens,
                       "parallelism": f"replicas x{world} (no collectives)", "prompt_mode": "accumulate",
                       "l2": "flushed (512 MiB write) before every step; inputs 154 MB per gamma > L2",
                       "cuda_graph": "one per gamma"},
            "per_gamma": per_gamma,
            "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                         "frac": round(achieved / peak, 4), "traffic": None,
                         "peak_source": f"{peak_src} bf16_tflops_sustained (burst {peak_burst})",
                         "frac_of_burst": round(achieved / peak_burst, 4),
                         "what": "whole forward: algorithmic FLOPs (SURVEY.md §8d F(model, gamma) x images) / device time"},
            "dominant_kernel": dom,
            "e2e": {"value": round(e2e_ips, 1), "unit": "images/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "how": "ServeModel.forward_async(pinned host fp32 images): H2D (copy stream) + forward + D2H logits per batch, next batch submitted before the previous is waited on; wall clock"},
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def dominant_gemm(cfg, B, dev, peak):
    """Times the fc1 GEMM (+bias+GELU epilogue) at the gamma = 0 shape alone with CUDA events."""
    from paper_2401_05031_b200 import _cuda

    lib = _cuda.lib()
    M, N, K = B * cfg.n_tokens, cfg.mlp_dim, cfg.dim
    a = torch.randn(M, K, device=dev).bfloat16()
    w = (torch.randn(N, K, device=dev) * 0.02).bfloat16()
    bias = torch.zeros(N, device=dev)
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    st = torch.cuda.current_stream(dev).cuda_stream
    for _ in range(5):
        _cuda.check(lib.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), None, out.data_ptr(), M, N, K, 1, 0, 0, st))
    n = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        _cuda.check(lib.ta_gemm(a.data_ptr(), w.data_ptr(), bias.data_ptr(), None, out.data_ptr(), M, N, K, 1, 0, 0, st))
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    tf = 2.0 * M * N * K / (ms / 1e3) / 1e12
    traffic = None  # DRAM bytes per launch from the committed `ncu --set full` capture of this shape
    try:
        import glob
        import re

        prof = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_gemm_fc1.txt")))[-1]
        vals = {k: float(v) for k, v in re.findall(r"(dram__bytes_(?:read|write)\.sum)\s+([0-9.]+)", open(prof).read())}
        traffic = {"bytes": round((vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]) * 1e6),
                   "algorithmic_bytes": 2 * (M * K + N * K + M * N), "source": os.path.basename(prof)}
    except Exception:
        pass
    return {"kernel": "gemm_bf16_sm100_pair_kernel<EPI_BIAS_GELU> (fc1 shape, timed alone via ta_gemm)", "shape": [M, N, K],
            "traffic": traffic,
            "ms": round(ms, 4), "achieved": round(tf, 1), "unit": "TFLOP/s", "peak": peak,
            "frac": round(tf / peak, 4), "bound": "tensor"}


def run_e2e(sm, cfg, B, gammas, args, dev):
    """Same metric end to end through the public API: pinned host images -> ServeModel.forward_async
    (H2D on a copy stream, forward, D2H of the logits) with the next batch submitted before the
    previous one is waited on, so copies overlap compute; every batch's logits reach the host."""
    imgs = {g: torch.randn(B, 3, cfg.img, cfg.img).pin_memory() for g in gammas}
    tasks = [0] * B
    for g in gammas:
        sm.forward_async(imgs[g], tasks, gamma=g).wait()
    steps = max(1, min(args.steps, 5))
    outs = [torch.empty(B, sm.backbone.max_classes).pin_memory() for _ in range(3)]
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    pending = []
    k = 0
    for _ in range(steps):
        for g in gammas:
            pending.append(sm.forward_async(imgs[g], tasks, gamma=g, out=outs[k % 3]))
            k += 1
            if len(pending) > 1:
                pending.pop(0).wait()  # at most two batches in flight (double-buffered slots)
    for p in pending:
        p.wait()
    dt = time.perf_counter() - t0
    h2d = len(gammas) * (B * 3 * cfg.img * cfg.img * 4 + B * 4)
    d2h = len(gammas) * B * sm.backbone.max_classes * 4
    return steps * len(gammas) * B / dt, h2d, d2h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="vit_b16")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--cpu-batch", type=int, default=8)
    ap.add_argument("--ref-batch", type=int, default=4)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--gammas", default="", help="comma-separated gamma sweep (default configs[1]: -16,-8,0,8,16)")
    ap.add_argument("--fold-ln", type=int, default=1, help="fold LayerNorm into the QKV / fc1 GEMMs (bf16 default)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
