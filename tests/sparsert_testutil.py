"""Shared test helpers (fixture loading, dtype rounding).  No method arithmetic."""
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def as_f16_f64(a) -> np.ndarray:
    """Round to IEEE fp16 (RN-even) and widen exactly to float64."""
    return np.asarray(a, dtype=np.float32).astype(np.float16).astype(np.float64)
