"""ServeModel front end on the GPU: per-task validation (only the tasks in the batch need a
head / prompts), id bounds at every gamma, errors naming the right task, ServeModel.execute,
and that the library leaves torch's current device alone."""

import pytest
import torch

from paper_2401_05031_b200.core import Batch, Query
from paper_2401_05031_b200.errors import ProfileGapError
from tests import helpers

pytestmark = pytest.mark.gpu


def _model():
    cfg, params = helpers.backbone("vit_tiny")
    tasks = helpers.task_params(cfg, (10, 100), [8])
    tasks[1]["prompts"] = {}  # task1 registered without prompts (INTEGRATION.md example)
    return cfg, params, tasks, helpers.serve_model(cfg, params, tasks, dtype="bf16")


def test_prompts_checked_per_task_in_batch():
    cfg, params, tasks, sm = _model()
    imgs = helpers.synthetic_images(4, cfg.img, seed=2)
    out = sm.forward(imgs.cuda(), ["task0"] * 4, gamma=8)  # task1 has no prompts: not in the batch
    torch.cuda.synchronize()
    ref, _ = helpers.oracle_forward(cfg, params, tasks, imgs, torch.zeros(4, dtype=torch.int64), 8)
    fin = torch.isfinite(ref)
    assert torch.isfinite(out.cpu()[fin]).all()
    assert (out.cpu()[fin] - ref[fin]).abs().max() <= 0.05 * ref[fin].abs().max()
    with pytest.raises(ProfileGapError) as ei:
        sm.forward(imgs.cuda(), ["task0", "task1", "task0", "task0"], gamma=8)
    assert ei.value.task == "task1" and ei.value.gamma == 8
    # the profiler skips the task without prompts at gamma 8 instead of failing
    table = sm.profile([0, 8], 4, iters=1, warmup=1)
    assert ("task0", 8) in table.sample_latency_us and ("task1", 8) not in table.sample_latency_us
    sm.backbone.close()


@pytest.mark.parametrize("gamma", [-4, 0, 8])
def test_task_id_bounds_every_gamma(gamma):
    cfg, params, tasks, sm = _model()
    imgs = helpers.synthetic_images(2, cfg.img, seed=2).cuda()
    for bad in ([0, 2], [-1, 0]):
        with pytest.raises(ValueError):
            sm.forward(imgs, torch.tensor(bad), gamma=gamma)
    sm.backbone.close()


def test_device_side_invalid_ids_give_nan_not_a_fault():
    """ta_forward with device ids cannot validate them on the host: an id out of range or a
    task without prompts yields NaN logits for that image only, never an illegal access."""
    cfg, params, tasks, sm = _model()
    bb = sm.backbone
    imgs = helpers.synthetic_images(3, cfg.img, seed=2).cuda()
    ids = torch.tensor([0, 7, 1], dtype=torch.int32, device="cuda")
    out = bb.forward_raw(imgs, ids, 8).cpu()
    torch.cuda.synchronize()
    assert torch.isfinite(out[0, :10]).all()
    assert torch.isnan(out[1]).all() and torch.isnan(out[2]).all()
    out0 = bb.forward_raw(imgs, ids, 0).cpu()
    assert torch.isfinite(out0[0, :10]).all() and torch.isfinite(out0[2, :100]).all()
    assert torch.isnan(out0[1]).all()
    # the context is still healthy
    assert torch.isfinite(bb.forward_raw(imgs, torch.zeros(3, dtype=torch.int32, device="cuda"), -4).cpu()[:, :10]).all()
    sm.backbone.close()


def test_execute_returns_latency_and_predictions():
    cfg, params, tasks, sm = _model()
    imgs = helpers.synthetic_images(5, cfg.img, seed=4)
    qs = [Query(i, "task0" if i % 2 == 0 else "task1", 0, 10_000, 1.0) for i in range(5)]
    payloads = {q.id: imgs[i] for i, q in enumerate(qs)}
    lat, preds = sm.execute(Batch(0, qs), -4, payloads)
    assert isinstance(lat, int) and lat > 0
    ref, _ = helpers.oracle_forward(cfg, params, tasks, imgs, torch.tensor([i % 2 for i in range(5)]), -4)
    for i, q in enumerate(qs):
        c = 10 if q.task == "task0" else 100
        assert 0 <= preds[i] < c
        top2 = ref[i, :c].topk(2).values
        if top2[0] - top2[1] > 0.05 * ref[i, :c].abs().max():
            assert preds[i] == int(ref[i, :c].argmax())
    sm.backbone.close()


def test_current_device_untouched():
    torch.cuda.set_device(0)
    cfg, params, tasks, sm = _model()
    assert torch.cuda.current_device() == 0
    sm.forward(helpers.synthetic_images(2, cfg.img).cuda(), [0, 0], gamma=0)
    assert torch.cuda.current_device() == 0
    sm.backbone.close()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_two_devices_one_process():
    """build_replicas(['cuda:0', 'cuda:1']) flow: each replica runs on its own device (the
    dynamic shared-memory attributes are set per device) and matches the other."""
    cfg, params = helpers.backbone("vit_tiny")
    tasks = helpers.task_params(cfg, (10,), [])
    from paper_2401_05031_b200.model import ServeModel, TaskModel, TransformerModel

    outs = []
    torch.cuda.set_device(0)
    for dev in ("cuda:0", "cuda:1"):
        bb = TransformerModel(cfg, params, dev, dtype="bf16", n_tasks=1, max_classes=10)
        sm = ServeModel(bb, [TaskModel("t", tasks[0]["head"]["w"], tasks[0]["head"]["b"], {})])
        imgs = helpers.synthetic_images(4, cfg.img, seed=1).to(dev)
        outs.append(sm.forward(imgs, [0] * 4, gamma=-4).cpu())
        assert torch.cuda.current_device() == 0
        bb.close()
    assert torch.equal(outs[0], outs[1])


def test_hf_checkpoint_end_to_end(tmp_path):
    """transformers ViTForImageClassification checkpoint -> from_hf_vit_state_dict -> GPU replica,
    head registered through a PromptRepository: logits match transformers' own forward of the
    same checkpoint (bf16 bound; fp32 mode rtol 1e-4)."""
    pytest.importorskip("transformers")
    from paper_2401_05031_b200.model import ServeModel, TransformerModel
    from paper_2401_05031_b200.repository import PromptRepository
    from paper_2401_05031_b200.weights import from_hf_vit_state_dict, head_from_hf_vit_state_dict
    from tests.golden.make_hf_golden import hf_model
    from tests.test_gpu_forward import BF16_TOL

    cfg, params = helpers.backbone("vit_tiny", seed=7)
    head = helpers.init_head(cfg, 10, 7)
    sd = hf_model(cfg, params, head).float().state_dict()
    repo = PromptRepository(str(tmp_path))
    h = head_from_hf_vit_state_dict(sd, cfg)
    repo.register_task("hf_task", h["w"], h["b"])
    imgs = helpers.synthetic_images(4, cfg.img, seed=9)
    with torch.no_grad():
        ref = hf_model(cfg, params, head).float()(pixel_values=imgs).logits
    for dtype, tol in (("fp32", 1e-4), ("bf16", BF16_TOL)):
        bb = TransformerModel(cfg, from_hf_vit_state_dict(sd, cfg), "cuda:0", dtype=dtype, n_tasks=1, max_classes=10)
        sm = ServeModel(bb)
        sm.register_from(repo)
        out = sm.forward(imgs.cuda(), ["hf_task"] * 4, gamma=0).cpu()
        scale = ref.abs().max().item()
        assert (out - ref).abs().max().item() <= tol * scale, dtype
        bb.close()
