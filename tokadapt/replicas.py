"""`tokadapt.replicas`: replica dispatch and throughput aggregation,
re-exported from paper_2401_05031_b200.replicas."""

from paper_2401_05031_b200.replicas import aggregate_throughput, earliest_free, round_robin  # noqa: F401

__all__ = ["round_robin", "earliest_free", "aggregate_throughput"]
