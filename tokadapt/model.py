"""`tokadapt.model`: the paper's serving entry points on the B200 path,
re-exported from paper_2401_05031_b200.model."""

from paper_2401_05031_b200.model import PendingForward, ServeModel, TaskModel, TransformerModel  # noqa: F401

__all__ = ["TransformerModel", "TaskModel", "ServeModel", "PendingForward"]
