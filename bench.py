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
Started as `python bench.py --gpus N` (no launcher), it re-launches itself as N ranks through
torch.distributed.run (replicas.launch_replicas).  --impl reference times the CPU oracle (the
reference has no implementation of the path; kind "port") on the host cores,
rank 0 only, one gamma of the sweep per step.
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


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


class CpuOracle:
    """The CPU reference of the path (oracle/vit_oracle.py, fp32 torch-CPU on all host threads):
    the reference ships no implementation of the forward, so this port is its
    CPU baseline.  Same seeded weights as the GPU replica (weights.py)."""

    def __init__(self, model: str, gammas):
        from paper_2401_05031_b200.config import VIT_CONFIGS
        from paper_2401_05031_b200.synthetic import synthetic_task_params
        from paper_2401_05031_b200.weights import init_backbone

        self.cfg = VIT_CONFIGS[model]
        self.params = init_backbone(self.cfg, 0)
        self.tasks = synthetic_task_params(self.cfg, (100,), [g for g in gammas if g > 0])
        self.cores = len(os.sched_getaffinity(0))
        torch.set_num_threads(self.cores)

    def run(self, batch: int, gamma: int, seed: int = 0) -> float:
        """Seconds for one forward of `batch` synthetic images at `gamma`."""
        from oracle import vit_oracle
        from paper_2401_05031_b200.weights import synthetic_images

        imgs = synthetic_images(batch, self.cfg.img, seed=seed)
        ids = torch.zeros(batch, dtype=torch.int64)
        heads = [t["head"] for t in self.tasks]
        prompts = [t["prompts"].get(gamma) for t in self.tasks] if gamma > 0 else None
        t0 = time.perf_counter()
        with torch.inference_mode():
            vit_oracle.forward(self.params, heads, imgs, ids, gamma, n_heads=self.cfg.heads,
                               patch=self.cfg.patch, prompts=prompts)
        return time.perf_counter() - t0


def cpu_baseline(model, gammas, batch, config1=True):
    """config 1 (b=8, gamma=-8) and one timed pass per gamma at the bench batch,
    on this box's host cores."""
    ora = CpuOracle(model, tuple(gammas) + ((-8,) if config1 else ()))
    ora.run(1, 0)  # warm-up (thread pool, allocator)
    out = {"unit": "images/s", "cores": ora.cores, "kind": "port", "cpu_model": cpu_model()}
    if config1:
        dt = ora.run(8, -8)
        out["config1"] = {"workload": f"{model} batch 8 gamma=-8 (configs[0])", "images_per_s": round(8 / dt, 3)}
    per, total_t = {}, 0.0
    for g in gammas:
        dt = ora.run(batch, g)
        per[str(g)] = round(batch / dt, 3)
        total_t += dt
    out["value"] = round(batch * len(gammas) / total_t, 3)
    out["per_gamma"] = per
    out["sample"] = (f"oracle/vit_oracle.py fp32 torch-CPU, one batch of {batch} per gamma {list(gammas)} "
                     f"({total_t:.1f} s){' + config 1' if config1 else ''}")
    return out


def run_reference(args):
    """--impl reference: the CPU reference of the path on the host cores (rank 0 only).  Each
    step is one batch of args.batch images at one gamma of the sweep, rotating through the
    gammas (a whole sweep at b=256 would take minutes per step); value = images / seconds."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    gammas = tuple(int(g) for g in args.gammas.split(",")) if args.gammas else GAMMAS
    ora = CpuOracle(args.model, gammas)
    for w in range(args.warmup):
        ora.run(1, gammas[w % len(gammas)], seed=100 + w)
    total_imgs, total_t, per = 0, 0.0, {}
    for s in range(args.steps):
        g = gammas[s % len(gammas)]
        dt = ora.run(args.batch, g, seed=s)
        total_imgs += args.batch
        total_t += dt
        per.setdefault(str(g), []).append(round(args.batch / dt, 3))
    value = total_imgs / total_t
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total_t / args.steps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": workload_config(args, gammas, args.gpus),
        "per_gamma": per,
        "cpu_baseline": {"value": round(value, 3), "unit": "images/s", "cores": ora.cores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"oracle/vit_oracle.py fp32 torch-CPU; step k = one batch of {args.batch} "
                                   f"at gamma {list(gammas)}[k mod {len(gammas)}], {args.steps} steps"},
        "e2e": {"value": round(value, 3), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, gammas, world):
    from paper_2401_05031_b200.config import VIT_CONFIGS

    cfg = VIT_CONFIGS[args.model]
    tag = " (configs[1])" if args.model == "vit_b16" and tuple(gammas) == GAMMAS and args.batch == 256 else ""
    return {"workload": f"{args.model} batch {args.batch} per gamma, sweep gamma in {list(gammas)}{tag}; one step = the sweep",
            "model": args.model, "global_batch": args.batch * len(gammas) * world, "seq_len": cfg.n_tokens,
            "parallelism": f"replicas x{world} (no collectives)", "prompt_mode": "accumulate",
            "l2": "flushed (512 MiB write) before every step; inputs 154 MB per gamma > L2",
            "cuda_graph": "one per gamma"}


def stage_bytes(cfg, gamma, B, fold_ln=True):
    """Algorithmic HBM bytes per forward of the memory-bound stages: patchify
    (read fp32 image, write bf16 patch matrix); the fused proj + merge of the merge layers (read
    the bf16 attention output and the fp32 residual, write every row once to its merged position
    (fp32) plus the kept rows' bf16 copy and row statistics, read the row map); merge_fixup
    (read / write the destination rows that received sources, read the source rows, sizes);
    match (read the k third of qkv, bf16; write the indices and the row map)."""
    from paper_2401_05031_b200.config import token_schedule

    D = cfg.dim
    ts, rs = token_schedule(cfg, gamma)
    patch = B * (3 * cfg.img * cfg.img * 4 + cfg.n_patches * cfg.patch_k_padded * 2)
    proj_merge = fixup = match = 0
    first = True
    for t, r in zip(ts, rs):
        if r <= 0:
            continue
        tp = t - r
        idx = (2 * r + (t + 1) // 2 - r) * 4
        proj_merge += B * (t * D * 2 + t * D * 4 + t * D * 4 + tp * D * 2 + tp * (D // 128) * 8 + t * 4)
        # at most r destinations: read + write x (fp32), write the bf16 copy and stats; r sources
        fixup += B * (r * D * 4 + r * (D * 4 + D * 4 + D * 2 + (D // 128) * 8) + (0 if first else t * 4) + tp * 4 + idx)
        match += B * (t * D * 2 + idx + t * 4)
        first = False
    return {"patchify": patch, "proj_merge": proj_merge, "fixup": fixup, "match": match}


def in_forward_profile(bb, cfg, B, dev, peak_burst, peak_sus, hbm_peak):
    """Stage times of eager forwards (ta_profile_stages: CUDA events on the forward's stream
    around every stage, kernels as the forward launches them), taken after a second of
    back-to-back forwards so the clocks are the power-capped ones of the timed region; median
    of 5 profiled forwards per gamma.  Gives the dominant kernel (fc1 = EPI_LN_GELU at gamma = 0,
    all 12 layers the same shape) and the achieved HBM bandwidth of the memory-bound stages."""
    imgs = torch.randn(B, 3, cfg.img, cfg.img, device=dev)
    ids = torch.zeros(B, dtype=torch.int32, device=dev)
    out = {}
    for g in (0, -8):
        t0 = time.time()
        while time.time() - t0 < 1.0:  # sustained load first: power-capped clocks
            for _ in range(10):
                bb.forward_raw(imgs, ids, g)
            torch.cuda.synchronize(dev)
        runs = [bb.stage_times(imgs, ids, g) for _ in range(5)]
        # per (stage, layer) position: the median over the runs
        out[g] = [(st, l, statistics.median(r[i][2] for r in runs)) for i, (st, l, _) in enumerate(runs[0])]
    fc1 = [us for st, l, us in out[0] if st == "fc1"]
    M, N, K = B * cfg.n_tokens, cfg.mlp_dim, cfg.dim
    us = sum(fc1) / len(fc1)
    tf = 2.0 * M * N * K / (us * 1e-6) / 1e12
    traffic = None
    try:
        import glob
        import re

        prof = sorted(glob.glob(os.path.join(ROOT, "profiles", "r02*_ncu_fc1_inforward.txt")))[-1]
        vals = {k: float(v) for k, v in re.findall(r"(dram__bytes_(?:read|write)\.sum)\s+([0-9.]+)", open(prof).read())}
        traffic = round((vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]) * 1e6)
    except Exception:
        pass
    # timed inside a forward after a second of sustained load (power-capped clocks): the
    # sustained peak is the denominator (B200_PROFILING.md), the burst one is reported beside it
    dom = {"kernel": "gemm_bf16_sm100_pair_kernel<EPI_LN_GELU> (fc1, in the gamma=0 forward)", "shape": [M, N, K],
           "us_per_launch": round(us, 2), "launches": len(fc1), "achieved": round(tf, 1), "unit": "TFLOP/s",
           "peak": peak_sus, "frac": round(tf / peak_sus, 4), "frac_of_burst": round(tf / peak_burst, 4),
           "bound": "tensor",
           "algorithmic_bytes": 2 * (M * K + N * K + M * N), "traffic": traffic,
           "how": "ta_profile_stages: CUDA events on the forward's stream around each fc1 launch (eager forwards "
                  "after 1 s of back-to-back forwards; median of 5)"}
    hbm = {}
    byts = stage_bytes(cfg, -8, B)
    ts, rs = __import__("paper_2401_05031_b200.config", fromlist=["token_schedule"]).token_schedule(cfg, -8)
    merge_layers = {l for l, r in enumerate(rs) if r > 0}
    times = {"patchify": sum(u for st, l, u in out[-8] if st == "patchify"),
             "proj_merge": sum(u for st, l, u in out[-8] if st == "proj" and l in merge_layers),
             "fixup": sum(u for st, l, u in out[-8] if st == "merge"),
             "match": sum(u for st, l, u in out[-8] if st == "match")}
    for nm, t_us in times.items():
        gbs = byts[nm] / (t_us * 1e-6) / 1e9
        hbm[nm] = {"gamma": -8, "bytes": byts[nm], "us": round(t_us, 1), "gbs": round(gbs, 1),
                   "frac": round(gbs / hbm_peak, 4)}
    stages0 = {}
    for st, l, u in out[0]:
        stages0[st] = round(stages0.get(st, 0.0) + u, 1)
    return dom, hbm, stages0


def run_ours(args):
    import torch.distributed as dist

    from paper_2401_05031_b200.config import VIT_CONFIGS, flops_per_image
    from paper_2401_05031_b200.replicas import aggregate_throughput
    from paper_2401_05031_b200.synthetic import build_serve_model

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")  # host-side plumbing only: barrier + reductions
    # one rank per GPU; if a box exposes fewer GPUs than ranks (multi-rank smoke tests on a
    # single-GPU box) ranks share devices round-robin
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    torch.cuda.set_device(dev)

    cfg = VIT_CONFIGS[args.model]
    gammas = tuple(int(g) for g in args.gammas.split(",")) if args.gammas else GAMMAS
    sm = build_serve_model(args.model, (100,), [g for g in gammas if g > 0], dtype="bf16", device=dev,
                           fold_ln=bool(args.fold_ln))
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

    def step():
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
        dist.barrier()  # barrier-aligned window on every replica
    torch.cuda.synchronize(dev)
    ev_list = []
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.steps):
            ev_list.append(step())
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    per_gamma_ms = {g: 0.0 for g in gammas}
    local_ms = 0.0
    for evs in ev_list:
        for i, g in enumerate(gammas):
            ms = evs[i].elapsed_time(evs[i + 1])
            per_gamma_ms[g] += ms
            local_ms += ms
    local_imgs = args.steps * len(gammas) * B
    # replicas only: images summed over ranks, device time = max over ranks
    imgs_total, total_ms = aggregate_throughput(local_imgs, local_ms)
    per_rank = [round(local_imgs / (local_ms / 1e3), 1)]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, {"rank": rank, "device": str(dev), "images_per_s": per_rank[0]})
        per_rank = gathered
    value = imgs_total / (total_ms / 1e3)
    peak_burst, peak_sus, hbm_peak, peak_src = _peaks()
    # the forward is timed inside a long step (tens of ms of back-to-back tensor work), so the
    # roofline denominator is the SUSTAINED bf16 figure; the burst one is reported beside it
    peak = peak_sus or peak_burst
    flops = {g: flops_per_image(cfg, g) for g in gammas}
    sweep_flops = sum(flops[g] * B for g in gammas) * args.steps
    achieved = sweep_flops / (local_ms / 1e3) / 1e12  # per GPU
    per_gamma = {}
    for g in gammas:
        ips = args.steps * B / (per_gamma_ms[g] / 1e3)
        tf = ips * flops[g] / 1e12
        per_gamma[str(g)] = {"images_per_s": round(ips, 1), "ms_per_batch": round(per_gamma_ms[g] / args.steps, 3),
                             "gflop_per_image": round(flops[g] / 1e9, 3), "tflops": round(tf, 1),
                             "roofline_frac": round(tf / peak, 4), "frac_of_burst": round(tf / peak_burst, 4)}

    # e2e through the public API: pinned host images -> ServeModel.forward_async -> host logits
    e2e_ips, h2d, d2h = run_e2e(sm, cfg, B, gammas, args, dev)
    if world > 1:
        t = torch.tensor([e2e_ips], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)  # slowest replica bounds the job
        e2e_ips = float(t.item()) * world

    dom, hbm, stages0 = in_forward_profile(bb, cfg, B, dev, peak_burst, peak_sus or peak_burst, hbm_peak)
    fp32_mode = None if args.no_fp32 else fp32_mode_line(args, cfg, gammas, B, dev)

    cpu = None
    if rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(args.model, gammas, args.cpu_batch)
    if world > 1:
        dist.barrier()  # other replicas wait while rank 0 times the CPU baseline

    launches = args.steps * sum(launches_per_forward(cfg, g, fold_ln=bool(args.fold_ln)) for g in gammas)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": workload_config(args, gammas, world),
            "per_gamma": per_gamma,
            "per_rank": per_rank,
            "roofline": {"bound": "tensor", "achieved": dom["achieved"], "peak": dom["peak"], "unit": "TFLOP/s",
                         "frac": dom["frac"], "frac_of_burst": dom["frac_of_burst"], "traffic": dom["traffic"],
                         "kernel": dom["kernel"],
                         "peak_source": f"{peak_src} bf16_tflops_sustained (the kernel runs inside a forward at power-capped clocks; burst {peak_burst})",
                         "forward": {"achieved": round(achieved, 1), "peak": peak, "frac": round(achieved / peak, 4),
                                     "peak_source": f"{peak_src} bf16_tflops_sustained (burst {peak_burst})",
                                     "frac_of_burst": round(achieved / peak_burst, 4),
                                     "what": "whole forward: algorithmic FLOPs (SURVEY.md §8d F(model, gamma) x images) / device time"}},
            "dominant_kernel": dom,
            "hbm": {"peak_gbs": hbm_peak, "stages": hbm,
                    "what": "algorithmic bytes (bench.stage_bytes) / stage device time in one eager forward, vs measured hbm_gbs"},
            "stages_gamma0_us": stages0,
            "e2e": {"value": round(e2e_ips, 1), "unit": "images/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "how": "ServeModel.forward_async(pinned host fp32 images): H2D (copy stream) + forward + D2H logits per batch, next batch submitted before the previous is waited on; wall clock"},
            "cpu_baseline": cpu,
            "fp32_mode": fp32_mode,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def fp32_mode_line(args, cfg, gammas, B, dev):
    """The same sweep in the fp32 parity mode (dtype="fp32": 3xTF32 tcgen05 GEMMs, fp32 attention /
    LayerNorm / merge, 3xTF32 matching), the precision of the paper's PyTorch prototype
    (PAPER.md:532-533): images/s per gamma, device time of 2 timed forwards after a warm-up."""
    from paper_2401_05031_b200.config import flops_per_image
    from paper_2401_05031_b200.synthetic import build_serve_model

    sm = build_serve_model(args.model, (100,), [g for g in gammas if g > 0], dtype="fp32", device=dev)
    bb = sm.backbone
    imgs = torch.randn(B, 3, cfg.img, cfg.img, device=dev)
    ids = torch.zeros(B, dtype=torch.int32, device=dev)
    per, tot_img, tot_ms = {}, 0, 0.0
    for g in gammas:
        bb.forward_raw(imgs, ids, g)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            bb.forward_raw(imgs, ids, g)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 2
        per[str(g)] = {"images_per_s": round(B / ms * 1e3, 1),
                       "tflops": round(flops_per_image(cfg, g) * B / ms / 1e9, 1)}
        tot_img += B
        tot_ms += ms
    bb.close()
    return {"value": round(tot_img / tot_ms * 1e3, 1), "unit": "images/s", "dtype": "fp32",
            "per_gamma": per, "gemm": "3xTF32 tcgen05 (kind::tf32, hi/lo split, chunked round-to-nearest accumulation)",
            "how": "one replica in fp32 parity mode, 2 forwards per gamma after a warm-up, CUDA events (not in the timed region)"}


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
    ap.add_argument("--cpu-batch", type=int, default=256, help="CPU baseline: images per gamma")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32 parity-mode summary")
    ap.add_argument("--gammas", default="", help="comma-separated gamma sweep (default configs[1]: -16,-8,0,8,16)")
    ap.add_argument("--fold-ln", type=int, default=1, help="fold LayerNorm into the QKV / fc1 GEMMs (bf16 default)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # started without a launcher: one process (replica) per GPU via torch.distributed.run
        from paper_2401_05031_b200.replicas import launch_replicas

        sys.exit(launch_replicas(args.gpus, os.path.abspath(__file__), sys.argv[1:]).returncode)
    run_ours(args)


if __name__ == "__main__":
    main()
