"""Parity metric of the reference (pkg/src/tvlp/oracle.py:228-234)."""
from __future__ import annotations

import numpy as np


def gradcheck_error(analytic, numeric):
    """Max elementwise deviation, normalized by the largest entry of either."""
    def _np(x):
        if hasattr(x, "detach"):
            x = x.detach().cpu().numpy()
        return np.asarray(x, dtype=np.float64)

    a, n = _np(analytic), _np(numeric)
    scale = max(np.max(np.abs(a), initial=0.0), np.max(np.abs(n), initial=0.0), 1e-8)
    return float(np.max(np.abs(a - n), initial=0.0) / scale)
