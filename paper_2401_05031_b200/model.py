"""ServeModel / TaskModel / TransformerModel — the paper's serving entry points
 on the B200 path.

* ``TransformerModel``: the shared ViT backbone with a prompt module before
  the norm and a merge module before the MLP in every layer; weights live on the GPU in
  the layouts of include/tokadapt_cuda.h.
* ``TaskModel``: per-task parameters = prompt tokens per gamma + head.
* ``ServeModel``: ``forward(inputs, tasks, task_params, gamma)`` over a
  mixed-task batch at one gamma; ``execute(batch, gamma, payloads)`` is the call an
  engine makes in place of ``estimate_batch`` (profiles.py:124); ``profile`` measures
  the (task, gamma) latency rows of profiles.py:82-121 on the device.

Every forward goes through libtokadapt_cuda.so (ctypes); there is no PyTorch or CPU
fallback for any stage of the path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple, Union

import torch

from . import _cuda
from .config import PROMPT_MODES, ViTConfig, token_schedule
from .core import Batch, us_from_s
from .errors import ConfigError, ProfileGapError
from .profiles import ProfileTable

__all__ = ["TransformerModel", "TaskModel", "ServeModel", "PendingForward"]

_DTYPES = {"bf16": _cuda.DTYPE_BF16, "fp32": _cuda.DTYPE_F32}


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class TransformerModel:
    """ViT backbone resident on one GPU.

    params: fp32 CPU master weights (weights.init_backbone layout, = timm state dict).
    dtype "bf16" runs the tcgen05 path; "fp32" is the parity mode (SIMT fp32 GEMMs).
    """

    def __init__(self, cfg: ViTConfig, params: Dict[str, object], device: Union[str, torch.device] = "cuda:0",
                 dtype: str = "bf16", prompt_mode: str = "accumulate", n_tasks: int = 1,
                 max_classes: int = 100, fold_ln: Optional[bool] = None):
        if dtype not in _DTYPES:
            raise ConfigError(f"dtype must be one of {sorted(_DTYPES)}")
        if prompt_mode not in PROMPT_MODES:
            raise ConfigError(f"prompt_mode must be one of {PROMPT_MODES}")
        self.cfg, self.dtype, self.prompt_mode = cfg, dtype, prompt_mode
        # bf16 mode folds LayerNorm into the QKV / fc1 GEMMs by default (fp32 parity mode
        # keeps the explicit LayerNorm passes): measured A/B (tools/ab_fold.py, ViT-B/16
        # b=256) -4% at gamma=-16, within +-1.5% elsewhere, -1% over the sweep
        self.fold_ln = (dtype == "bf16") if fold_ln is None else bool(fold_ln and dtype == "bf16")
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise ConfigError("TransformerModel runs on a CUDA device only (no CPU fallback)")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.n_tasks, self.max_classes = n_tasks, max_classes
        self._lib = _cuda.lib()
        desc = _cuda.ModelDesc(cfg.dim, cfg.depth, cfg.heads, cfg.mlp_dim, cfg.patch, cfg.img,
                               n_tasks, max_classes,
                               _cuda.PROMPT_ACCUMULATE if prompt_mode == "accumulate" else _cuda.PROMPT_REPLACE,
                               _DTYPES[dtype])
        handle = ctypes.c_void_p()
        _cuda.check(self._lib.ta_model_create(self.device.index, ctypes.byref(desc), ctypes.byref(handle)))
        self._h = handle
        self._keep: List[torch.Tensor] = []
        self._upload(params)
        self._ws: Dict[Tuple[int, int], torch.Tensor] = {}

    # -- weights -------------------------------------------------------------------
    def _mat(self, w: torch.Tensor) -> torch.Tensor:
        dt = torch.bfloat16 if self.dtype == "bf16" else torch.float32
        t = w.to(device=self.device, dtype=dt).contiguous()
        self._keep.append(t)
        return t

    def _vec(self, v: torch.Tensor) -> torch.Tensor:
        t = v.to(device=self.device, dtype=torch.float32).contiguous()
        self._keep.append(t)
        return t

    def _upload(self, p: Dict[str, object]) -> None:
        cfg = self.cfg
        pw = p["patch_w"].reshape(cfg.dim, cfg.patch_k)
        if cfg.patch_k_padded != cfg.patch_k:
            pw = torch.nn.functional.pad(pw, (0, cfg.patch_k_padded - cfg.patch_k))
        layers = (_cuda.LayerWeights * cfg.depth)()
        for i, lw in enumerate(p["layers"]):
            vals = {}
            for k in ("qkv_w", "proj_w", "fc1_w", "fc2_w"):
                vals[k] = _ptr(self._mat(lw[k]))
            for k in ("ln1_w", "ln1_b", "qkv_b", "proj_b", "ln2_w", "ln2_b", "fc1_b", "fc2_b"):
                vals[k] = _ptr(self._vec(lw[k]))
            if self.fold_ln:
                # LayerNorm folded into the following GEMM (include/tokadapt_cuda.h):
                # W' = bf16(W o gamma), c1 = rowsum(W') (of the rounded values), c2 = W beta + b
                for name, ln in (("qkv", "ln1"), ("fc1", "ln2")):
                    w32 = lw[f"{name}_w"].double()
                    wf = (w32 * lw[f"{ln}_w"].double()[None, :]).to(torch.bfloat16)
                    vals[f"{name}_w_ln"] = _ptr(self._mat(wf))
                    vals[f"{name}_c1"] = _ptr(self._vec(wf.double().sum(dim=1).float()))
                    c2 = w32 @ lw[f"{ln}_b"].double() + lw[f"{name}_b"].double()
                    vals[f"{name}_c2"] = _ptr(self._vec(c2.float()))
            layers[i] = _cuda.LayerWeights(**vals)
        self._layers_c = layers
        self._weights_c = _cuda.Weights(
            _ptr(self._mat(pw)), _ptr(self._vec(p["patch_b"])), _ptr(self._vec(p["cls"])),
            _ptr(self._vec(p["pos"])), _ptr(self._vec(p["norm_w"])), _ptr(self._vec(p["norm_b"])),
            ctypes.cast(layers, ctypes.POINTER(_cuda.LayerWeights)))
        _cuda.check(self._lib.ta_model_set_weights(self._h, ctypes.byref(self._weights_c)))

    def set_head(self, task: int, w: torch.Tensor, b: torch.Tensor) -> None:
        wt, bt = self._vec(w), self._vec(b)
        _cuda.check(self._lib.ta_model_set_head(self._h, task, wt.data_ptr(), bt.data_ptr(), int(w.shape[0])))

    def set_prompts(self, task: int, gamma: int, prompts: torch.Tensor) -> None:
        cfg = self.cfg
        if tuple(prompts.shape) != (cfg.depth, gamma, cfg.dim):
            raise ValueError(f"prompts must be [L={cfg.depth}, gamma={gamma}, D={cfg.dim}]")
        pt = self._vec(prompts)
        _cuda.check(self._lib.ta_model_set_prompts(self._h, task, gamma, pt.data_ptr()))

    # -- schedule / workspace --------------------------------------------------------
    def schedule(self, gamma: int) -> Tuple[List[int], List[int]]:
        return token_schedule(self.cfg, gamma, self.prompt_mode)

    def workspace(self, batch: int, gamma: int) -> torch.Tensor:
        key = (batch, gamma)
        ws = self._ws.get(key)
        if ws is None:
            n = ctypes.c_size_t()
            _cuda.check(self._lib.ta_workspace_size(self._h, batch, gamma, ctypes.byref(n)))
            ws = torch.empty(n.value, dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def trace_len(self, batch: int, gamma: int) -> int:
        n = ctypes.c_size_t()
        _cuda.check(self._lib.ta_merge_trace_len(self._h, batch, gamma, ctypes.byref(n)))
        return n.value

    # -- forward -------------------------------------------------------------------
    def forward_raw(self, images: torch.Tensor, task_ids: torch.Tensor, gamma: int,
                    logits: Optional[torch.Tensor] = None, trace: Optional[torch.Tensor] = None,
                    forced_trace: Optional[torch.Tensor] = None,
                    workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Device tensors in, device logits out; asynchronous on the current stream."""
        b = images.shape[0]
        if images.dtype != torch.float32 or not images.is_contiguous() or images.device != self.device:
            raise ValueError("images must be contiguous fp32 on the model's device")
        if task_ids.dtype != torch.int32 or task_ids.device != self.device:
            raise ValueError("task ids must be int32 on the model's device")
        if logits is None:
            logits = torch.empty(b, self.max_classes, dtype=torch.float32, device=self.device)
        ws = workspace if workspace is not None else self.workspace(b, gamma)
        # the library switches to (and restores) the model's device itself; the stream is the
        # current stream of the model's device
        rc = self._lib.ta_forward(self._h, images.data_ptr(), task_ids.data_ptr(), b, gamma,
                                  logits.data_ptr(), _ptr(trace), _ptr(forced_trace),
                                  ws.data_ptr(), ws.numel(), _stream_handle(self.device))
        _cuda.check(rc, gamma=gamma)
        return logits

    def forward_host(self, images: torch.Tensor, task_ids: torch.Tensor, gamma: int,
                     out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Host (CPU, ideally pinned) tensors in and out through ta_forward_host."""
        b = images.shape[0]
        imgs = images.contiguous()
        tids = task_ids.to(torch.int32).contiguous()
        if out is None:
            out = torch.empty(b, self.max_classes, dtype=torch.float32)
        rc = self._lib.ta_forward_host(self._h, imgs.data_ptr(), tids.data_ptr(), b, gamma,
                                       out.data_ptr(), _stream_handle(self.device))
        _cuda.check(rc, gamma=gamma)
        return out

    def forward_host_async(self, images: torch.Tensor, task_ids: torch.Tensor, gamma: int,
                           out: Optional[torch.Tensor] = None) -> "PendingForward":
        """Pipelined host path: pinned host images -> device (copy stream, one of two staging
        slots) -> forward on the model's current stream -> logits back into the pinned
        ``out``; returns at once with a handle (``wait()`` -> logits).  Consecutive calls overlap
        the next batch's H2D with the current forward, so a stream of host batches runs at the
        device rate instead of copy + compute + copy in series."""
        b = images.shape[0]
        if images.dtype != torch.float32 or images.device.type != "cpu":
            raise ValueError("images must be fp32 host tensors (pinned for overlap)")
        if out is None:
            out = torch.empty(b, self.max_classes, dtype=torch.float32, pin_memory=True)
        if not hasattr(self, "_copy_stream"):
            self._copy_stream = torch.cuda.Stream(self.device)
            self._slots: List[Dict[str, object]] = [{}, {}]
            self._slot_k = 0
        slot = self._slots[self._slot_k & 1]
        self._slot_k += 1
        shape = tuple(images.shape)
        if slot.get("shape") != shape:
            slot.update(shape=shape, img=torch.empty(shape, dtype=torch.float32, device=self.device),
                        ids=torch.empty(b, dtype=torch.int32, device=self.device),
                        logits=torch.empty(b, self.max_classes, dtype=torch.float32, device=self.device),
                        free=None)
        compute = torch.cuda.current_stream(self.device)
        with torch.cuda.stream(self._copy_stream):
            if slot["free"] is not None:  # the forward that last read this slot is done
                self._copy_stream.wait_event(slot["free"])
            slot["img"].copy_(images, non_blocking=True)
            slot["ids"].copy_(task_ids.to(torch.int32), non_blocking=True)
            h2d = torch.cuda.Event()
            h2d.record(self._copy_stream)
        compute.wait_event(h2d)
        self.forward_raw(slot["img"], slot["ids"], gamma, logits=slot["logits"])
        free = torch.cuda.Event()
        free.record(compute)
        slot["free"] = free
        out.copy_(slot["logits"], non_blocking=True)
        done = torch.cuda.Event()
        done.record(compute)
        return PendingForward(done, out)

    def stage_times(self, images: torch.Tensor, task_ids: torch.Tensor, gamma: int) -> List[Tuple[str, int, float]]:
        """One eager forward with per-stage CUDA events (ta_profile_stages): returns
        [(stage, layer, device us)] in launch order (layer -1 = outside the layer loop).
        Synchronises; not for use inside a CUDA graph."""
        _cuda.check(self._lib.ta_profile_stages(self._h, 1))
        try:
            self.forward_raw(images, task_ids, gamma)
            torch.cuda.synchronize(self.device)
            n = ctypes.c_int()
            _cuda.check(self._lib.ta_stage_records(self._h, None, 0, ctypes.byref(n)))
            recs = (_cuda.StageRecord * max(1, n.value))()
            _cuda.check(self._lib.ta_stage_records(self._h, recs, n.value, ctypes.byref(n)))
        finally:
            _cuda.check(self._lib.ta_profile_stages(self._h, 0))
        return [(_cuda.STAGES[r.stage], r.layer, float(r.us)) for r in recs[:n.value]]

    def close(self) -> None:
        if getattr(self, "_h", None):
            torch.cuda.synchronize(self.device)
            self._lib.ta_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class PendingForward:
    """Handle of ``forward_host_async``: ``wait()`` blocks until the logits are on the host."""

    event: object
    logits: torch.Tensor

    def wait(self) -> torch.Tensor:
        self.event.synchronize()
        return self.logits


@dataclass
class TaskModel:
    """Per-task parameters: head [C, D] + prompts per gamma [L, gamma, D]."""

    name: str
    head_w: torch.Tensor
    head_b: torch.Tensor
    prompts: Dict[int, torch.Tensor] = field(default_factory=dict)

    @property
    def classes(self) -> int:
        return int(self.head_w.shape[0])


class ServeModel:
    """Front end over one backbone replica and its registered tasks."""

    def __init__(self, backbone: TransformerModel, tasks: Sequence[TaskModel] = ()):
        self.backbone = backbone
        self.tasks: List[TaskModel] = []
        self.task_index: Dict[str, int] = {}
        for t in tasks:
            self.register_task(t)

    def register_task(self, task: TaskModel) -> int:
        """Register_Task: head + prompt repository entries."""
        if task.name in self.task_index:
            raise ConfigError(f"task {task.name!r} already registered")
        idx = len(self.tasks)
        if idx >= self.backbone.n_tasks:
            raise ConfigError(f"backbone was built for {self.backbone.n_tasks} tasks")
        if task.classes > self.backbone.max_classes:
            raise ConfigError(f"task {task.name!r} has {task.classes} classes > max_classes")
        self.backbone.set_head(idx, task.head_w, task.head_b)
        for gamma, p in task.prompts.items():
            self.backbone.set_prompts(idx, gamma, p)
        self.tasks.append(task)
        self.task_index[task.name] = idx
        return idx

    def register_from(self, repo, tasks: Optional[Sequence[str]] = None,
                      gammas: Optional[Sequence[int]] = None) -> List[int]:
        """Register tasks of a ``PromptRepository`` (all by default) with this replica: heads and
        the prompts for ``gammas`` (default: every stored gamma).  Returns their task ids."""
        return [self.register_task(repo.task_model(t, list(gammas) if gammas is not None else None))
                for t in (tasks if tasks is not None else repo.tasks())]

    def task_ids(self, tasks: Union[Sequence[str], Sequence[int], torch.Tensor]) -> torch.Tensor:
        if isinstance(tasks, torch.Tensor):
            ids = tasks.to(torch.int32)
        else:
            ids = torch.tensor([self.task_index[t] if isinstance(t, str) else int(t) for t in tasks],
                               dtype=torch.int32)
        return ids

    def _check_gamma(self, ids_host: torch.Tensor, gamma: int) -> None:
        """Validate the batch's task ids (every gamma: an id indexes the device head / prompt
        tables) and, for gamma > 0, that each task in the batch has prompts at gamma
        (ProfileGapError names the task, as the reference's prompt lookup does)."""
        if gamma < -(self.backbone.cfg.n_tokens - 1):
            raise ValueError(f"gamma {gamma} merges more tokens than exist")
        for i in set(ids_host.tolist()):
            if i < 0 or i >= len(self.tasks):
                raise ValueError(f"unknown task id {i}")
            if gamma > 0 and gamma not in self.tasks[i].prompts:
                raise ProfileGapError(self.tasks[i].name, gamma, "prompt")

    def forward(self, inputs: torch.Tensor, tasks, task_params=None, gamma: int = 0) -> torch.Tensor:
        """ServeModel.forward(inputs, tasks, task_params, gamma).

        inputs [B, 3, S, S] fp32 (device or host); tasks = names / ids / int tensor;
        task_params (optional) TaskModels to register first.  Returns logits
        [B, max_classes] on the inputs' device, -inf beyond each task's class count.
        """
        if task_params:
            for tp in task_params:
                if tp.name not in self.task_index:
                    self.register_task(tp)
        ids = self.task_ids(tasks)
        self._check_gamma(ids.cpu(), gamma)
        with torch.cuda.device(self.backbone.device):
            if inputs.device.type == "cpu":
                return self.backbone.forward_host(inputs.float(), ids, gamma)
            return self.backbone.forward_raw(inputs.float().contiguous(), ids.to(self.backbone.device), gamma)

    __call__ = forward

    def forward_async(self, inputs: torch.Tensor, tasks, gamma: int = 0,
                      out: Optional[torch.Tensor] = None) -> PendingForward:
        """Host-batch pipelining over ``TransformerModel.forward_host_async``: returns at once;
        ``.wait()`` gives the host logits.  Submitting the next batch before waiting overlaps
        its H2D copy with the current forward."""
        ids = self.task_ids(tasks)
        self._check_gamma(ids.cpu(), gamma)
        with torch.cuda.device(self.backbone.device):
            return self.backbone.forward_host_async(inputs.float(), ids, gamma, out=out)

    def execute(self, batch: Batch, gamma: int, payloads: Dict[int, torch.Tensor]) -> Tuple[int, List[int]]:
        """Run a planned batch (engine step) and return (latency_us, predictions).

        payloads maps query id -> image [3, S, S]; Batch itself carries metadata only
        (SPEC.md:90).  Latency is device time (CUDA events) in integer microseconds, the
        unit of the whole scheduler (core.py:3-5).
        """
        imgs = torch.stack([payloads[q.id] for q in batch.queries]).to(self.backbone.device, torch.float32)
        ids = self.task_ids([q.task for q in batch.queries])
        self._check_gamma(ids, gamma)
        dev = self.backbone.device
        with torch.cuda.device(dev):
            ids_dev = ids.to(dev)
            stream = torch.cuda.current_stream(dev)
            start = torch.cuda.Event(enable_timing=True)
            end = torch.cuda.Event(enable_timing=True)
            start.record(stream)
            logits = self.backbone.forward_raw(imgs.contiguous(), ids_dev, gamma)
            end.record(stream)
            end.synchronize()
        latency_us = us_from_s(start.elapsed_time(end) / 1e3)
        preds = []
        for i, q in enumerate(batch.queries):
            c = self.tasks[self.task_index[q.task]].classes
            preds.append(int(logits[i, :c].argmax().item()))
        return latency_us, preds

    def profile(self, gammas: Sequence[int], batch_size: int, accuracy: Optional[Dict[Tuple[str, int], float]] = None,
                iters: int = 5, warmup: int = 2, seed: int = 0) -> ProfileTable:
        """B200 task profiler: measure per-sample and
        per-batch latency for every registered task at each gamma and return a
        ProfileTable (write it with profiles.write_profile_csv)."""
        table = ProfileTable(base_tokens=self.backbone.cfg.n_tokens, layers=self.backbone.cfg.depth)
        cfg = self.backbone.cfg
        dev = self.backbone.device
        g = torch.Generator(device=dev).manual_seed(seed)
        imgs = torch.randn(batch_size, 3, cfg.img, cfg.img, generator=g, device=dev)
        with torch.cuda.device(dev):
            return self._profile(table, imgs, gammas, batch_size, accuracy, iters, warmup)

    def _profile(self, table, imgs, gammas, batch_size, accuracy, iters, warmup) -> ProfileTable:
        dev = self.backbone.device
        stream = torch.cuda.current_stream(dev)
        for gamma in gammas:
            batch_times = []
            for ti, task in enumerate(self.tasks):
                if gamma > 0 and gamma not in task.prompts:
                    continue
                ids = torch.full((batch_size,), ti, dtype=torch.int32, device=dev)
                for _ in range(warmup):
                    self.backbone.forward_raw(imgs, ids, gamma)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                for _ in range(iters):
                    self.backbone.forward_raw(imgs, ids, gamma)
                e.record(stream)
                e.synchronize()
                sec = s.elapsed_time(e) / 1e3 / iters
                batch_times.append(sec)
                table.sample_latency_us[(task.name, gamma)] = max(1, us_from_s(sec / batch_size))
                table.accuracy[(task.name, gamma)] = (accuracy or {}).get((task.name, gamma), 1.0)
            if batch_times:
                table.batch_latency_us[(gamma, batch_size)] = max(1, us_from_s(sum(batch_times) / len(batch_times)))
        return table
