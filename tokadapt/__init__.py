"""Drop-in import name of the reference package (pkg/pyproject.toml: dist `tokadapt`).

`import tokadapt.core` / `tokadapt.profiles` / `tokadapt.errors` resolve to the B200
implementation in paper_2401_05031_b200; `tokadapt.model` (ServeModel / TaskModel /
TransformerModel) and `tokadapt.replicas` are real submodules (so
`from tokadapt.model import ServeModel` works) that load the CUDA library lazily;
`tokadapt.batcher` / `adapter` / `workload` / `engine` are the SPEC.md serving modules
(Alg. 1-3, workloads, engine + metrics)."""

import sys as _sys

from paper_2401_05031_b200 import adapter, batcher, config, core, engine, errors, profiles, weights, workload  # noqa: F401

for _name in ("core", "errors", "profiles", "config", "weights", "batcher", "adapter", "workload", "engine"):
    _sys.modules[f"{__name__}.{_name}"] = getattr(_sys.modules["paper_2401_05031_b200"], _name)
