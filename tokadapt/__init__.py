"""Drop-in import name of the reference package (pkg/pyproject.toml: dist `tokadapt`).

`import tokadapt.core` / `tokadapt.profiles` / `tokadapt.errors` resolve to the B200
implementation in paper_2401_05031_b200; `tokadapt.model` adds ServeModel / TaskModel /
TransformerModel."""

import sys as _sys

from paper_2401_05031_b200 import config, core, errors, profiles, weights  # noqa: F401

for _name in ("core", "errors", "profiles", "config", "weights"):
    _sys.modules[f"{__name__}.{_name}"] = getattr(_sys.modules["paper_2401_05031_b200"], _name)


def __getattr__(name):
    if name in ("model", "_cuda", "serving"):
        import importlib

        mod = importlib.import_module(f"paper_2401_05031_b200.{name}")
        _sys.modules[f"{__name__}.{name}"] = mod
        return mod
    raise AttributeError(name)
