"""Generates the committed golden fixtures under tests/golden/.

  host_api_kats.json   outputs of the REFERENCE host API (pkg/src/tokadapt/{core,profiles,
                       errors}.py), imported from /root/reference under an alias package
                       name, on the SPEC's worked examples and on seeded random cases.  These
                       pin our re-implementation (paper_2401_05031_b200.core / .profiles).
  oracle_tiny.npz      oracle/vit_oracle.py forward of the seeded ViT-tiny configuration for
                       several gammas (logits + merge traces): freezes the oracle so later
                       edits cannot drift silently (the path itself is parity-unpinned, see
                       oracle/vit_oracle.py).
  oracle_b16_cfg1.npz  config 1 of BASELINE.json: ViT-B/16, batch 8, gamma = -8, fp32 and fp64.

Run from the repo root in a container that has /root/reference:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import importlib.util
import json
import os
import random
import sys
import tempfile

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src/tokadapt"


def load_reference(alias: str = "tokadapt_ref"):
    """Import the reference package as `alias` so it cannot shadow anything of ours."""
    spec = importlib.util.spec_from_file_location(alias, os.path.join(REF_SRC, "__init__.py"),
                                                  submodule_search_locations=[REF_SRC])
    if spec is None or not os.path.isdir(REF_SRC):
        raise RuntimeError("reference not available")
    # tokadapt is a namespace package (no __init__.py): build the package module by hand
    import types

    pkg = types.ModuleType(alias)
    pkg.__path__ = [REF_SRC]
    sys.modules[alias] = pkg
    mods = {}
    for name in ("errors", "core", "profiles"):
        s = importlib.util.spec_from_file_location(f"{alias}.{name}", os.path.join(REF_SRC, f"{name}.py"))
        m = importlib.util.module_from_spec(s)
        sys.modules[f"{alias}.{name}"] = m
        s.loader.exec_module(m)
        mods[name] = m
    return mods


def host_api_cases(ref) -> dict:
    core, prof, err = ref["core"], ref["profiles"], ref["errors"]
    out: dict = {}
    # --- core: SPEC.md:59-61 batch_attributes examples and random batches
    cases = []
    rng = random.Random(0)
    specs = [
        [(1, "A", 1_000_000, 600_000, 0.3), (2, "B", 1_200_000, 400_000, 0.5)],
        [(7, "A", 5_000_000, 600_000, 1.0), (8, "A", 5_000_000, 700_000, 2.0)],
    ]
    for _ in range(20):
        n = rng.randint(1, 6)
        specs.append([(rng.randint(0, 50), rng.choice("ABC"), rng.randint(0, 10) * 100_000,
                       rng.randint(1, 9) * 100_000, round(rng.random(), 3)) for _ in range(n)])
    for sp in specs:
        qs = [core.Query(*q) for q in sp]
        b = core.Batch(0, qs)
        cases.append({"queries": sp, "attributes": list(core.batch_attributes(b)),
                      "incremental": [b.arrival_us, b.deadline_us, b.anchor_utility,
                                      b.max_deadline_gap_at_admission_us,
                                      b.max_utility_gap_at_admission],
                      "task_counts": b.task_counts, "task_utility": b.task_utility})
    out["batches"] = cases
    # classify_outcome
    q = core.Query(1, "A", 0, 100, 1.0)
    out["classify"] = [[f, c, t, core.classify_outcome(q, f, c, t).value]
                       for f in (True, False) for c in (True, False) for t in (50, 99, 100, 150)]
    out["us_from_s"] = [[s, core.us_from_s(s)] for s in (0.0, 1e-6, 0.0000015, 0.0000025, 1.5, 1 / 300)]
    # --- profiles: SPEC.md:126-138 examples
    table = prof.ProfileTable(accuracy={("A", 2): 0.5, ("B", 2): 0.5},
                              sample_latency_us={("A", 2): 2000, ("B", 2): 3000})
    b = core.Batch(0, [core.Query(i, "A", 0, 1000, 1.0) for i in range(3)] +
                   [core.Query(10 + i, "B", 0, 1000, 2.0) for i in range(2)])
    out["estimate_batch"] = list(prof.estimate_batch(b, 2, table))
    mem = prof.MemoryModel(c0_bytes=0, c1_bytes_per_token=1, gpu_capacity_bytes=1 << 30)
    mt = prof.ProfileTable(base_tokens=197, layers=12)
    bb = core.Batch(0, [core.Query(0, "A", 0, 10, 1.0)])
    out["batch_memory"] = [[g, prof.batch_memory(bb, g, mem, mt)] for g in (-16, -8, 0, 8, 16, 49)]
    rmap = prof.RateToGammaMap(((0.0, 8), (280.0, 4), (320.0, 2), (350.0, 0), (380.0, -5),
                                (450.0, -10), (520.0, -15), (1000.0, -20)))
    out["project_rate"] = [[r, prof.project_rate(r, rmap)] for r in
                           (0, 279, 280, 319, 320, 349, 350, 380, 450, 520, 999, 1000, 1200)]
    gl = core.GammaList((-20, -15, -10, -5, 0, 2, 4, 8))
    dt = prof.ProfileTable()
    for i, g in enumerate(gl):
        dt.sample_latency_us[("A", g)] = 1000 + 300 * i
        dt.accuracy[("A", g)] = 0.5 + 0.05 * i
    out["derive_f"] = [list(p) for p in prof.derive_f(dt, gl, 8).breakpoints]
    # CSV round trip + error messages
    with tempfile.TemporaryDirectory() as d:
        good = os.path.join(d, "p.csv")
        with open(good, "w") as fh:
            fh.write("kind,task,gamma,batch_size,value\n"
                     "accuracy,A,0,,0.9\nsample_latency_s,A,0,,0.002\nsample_latency_s,A,4,,0.003\n"
                     "accuracy,A,4,,0.95\nbatch_latency_s,A,0,8,0.01\n\n")
        t = prof.load_profile_csv(good)
        out["csv"] = {"accuracy": [[k[0], k[1], v] for k, v in sorted(t.accuracy.items())],
                      "sample": [[k[0], k[1], v] for k, v in sorted(t.sample_latency_us.items())],
                      "batch": [[k[0], k[1], v] for k, v in sorted(t.batch_latency_us.items())]}
        errs = {}
        for name, body in {
            "header": "kind,task,gamma\naccuracy,A,0\n",
            "columns": "kind,task,gamma,batch_size,value\naccuracy,A,0\n",
            "kind": "kind,task,gamma,batch_size,value\nfoo,A,0,,1\n",
            "monotone": "kind,task,gamma,batch_size,value\nsample_latency_s,A,0,,0.003\nsample_latency_s,A,4,,0.002\n",
            "number": "kind,task,gamma,batch_size,value\naccuracy,A,x,,1\n",
            "accuracy_range": "kind,task,gamma,batch_size,value\naccuracy,A,0,,1.5\n",
        }.items():
            p = os.path.join(d, name + ".csv")
            with open(p, "w") as fh:
                fh.write(body)
            try:
                prof.load_profile_csv(p)
                errs[name] = None
            except Exception as e:  # noqa: BLE001
                errs[name] = [type(e).__name__, str(e).replace(p, "<path>")]
        out["csv_errors"] = errs
    out["gap_error"] = str(err.ProfileGapError("A", 4, "prompt"))
    return out


def oracle_goldens() -> None:
    from oracle import vit_oracle  # noqa: F401
    from tests import helpers

    cfg, params = helpers.backbone("vit_tiny")
    data = {}
    for gamma in (-8, -4, -1, 0, 2, 8):
        tasks = helpers.task_params(cfg, (10, 100), [gamma] if gamma > 0 else [])
        imgs = helpers.synthetic_images(6, cfg.img, seed=0)
        ids = torch.arange(6) % 2
        for mode in (("accumulate", "replace") if gamma > 0 else ("accumulate",)):
            logits, tr = helpers.oracle_forward(cfg, params, tasks, imgs, ids, gamma, mode)
            key = f"g{gamma}_{mode}"
            data[key + "_logits"] = logits.numpy()
            data[key + "_trace"] = tr.flat_int32().numpy()
    np.savez_compressed(os.path.join(HERE, "oracle_tiny.npz"), **data)

    cfg, params = helpers.backbone("vit_b16")
    tasks = helpers.task_params(cfg, (10, 100), [])
    imgs = helpers.synthetic_images(8, cfg.img, seed=0)
    ids = torch.arange(8) % 2
    l32, t32 = helpers.oracle_forward(cfg, params, tasks, imgs, ids, -8)
    l64, t64 = helpers.oracle_forward(cfg, params, tasks, imgs, ids, -8, dtype=torch.float64)
    margins = np.array([float((m.node_max.sort(dim=-1, descending=True).values[:, m.r - 1] -
                               m.node_max.sort(dim=-1, descending=True).values[:, m.r]).min())
                        for m in t64.merges])
    np.savez_compressed(os.path.join(HERE, "oracle_b16_cfg1.npz"), logits32=l32.numpy(),
                        logits64=l64.numpy(), trace32=t32.flat_int32().numpy(),
                        trace64=t64.flat_int32().numpy(), topr_gap_fp64=margins)


if __name__ == "__main__":
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    ref = load_reference()
    with open(os.path.join(HERE, "host_api_kats.json"), "w") as fh:
        json.dump(host_api_cases(ref), fh, indent=1, sort_keys=True)
    oracle_goldens()
    print("wrote", sorted(os.listdir(HERE)))
