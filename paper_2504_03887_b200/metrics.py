"""The one metric on the estimation path (metrics.py:91-95); the paper's
evaluation metrics are out of scope."""

from __future__ import annotations


def predict_oom(predicted_peak: int, capacity: int) -> bool:
    """A job is predicted to OOM when its peak strictly exceeds capacity."""
    if predicted_peak <= 0 or capacity <= 0:
        raise ValueError("predicted_peak and capacity must be positive")
    return predicted_peak > capacity
