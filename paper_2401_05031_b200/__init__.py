"""B200-native token-adapted ViT inference (OTAS, arXiv 2401.05031).

Host API (drop-in for the reference's ``tokadapt`` package): ``core``, ``profiles``,
``errors`` mirror pkg/src/tokadapt/*.py; ``model`` adds the paper's ServeModel /
TaskModel / TransformerModel on top of the sm_100a CUDA library (``_cuda``); ``batcher``,
``adapter``, ``workload`` and ``engine`` are the host-side serving loop (Alg. 1-3) that plans
gamma per batch and executes it on GPU replicas.
"""

from . import adapter, batcher, config, core, engine, errors, profiles, weights, workload  # noqa: F401
from .config import VIT_CONFIGS, ViTConfig, flops_per_image, token_schedule  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # model / _cuda load the CUDA library lazily so that the host API imports without a GPU.
    if name in ("model", "_cuda"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    if name in ("ServeModel", "TaskModel", "TransformerModel"):
        from . import model

        return getattr(model, name)
    raise AttributeError(name)
