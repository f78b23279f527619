"""B200-native differentiable sample-wise linear prediction (arXiv 2406.05128).

Drop-in for the LP path of the reference ``tvlp`` 0.1.0 package: the
``tvlp.lpc`` functional API (``lp_forward_tv``, ``lp_backward_tv``,
``lp_forward_ti``, ``lp_backward_ti``, ``shift_coeffs``,
``lagged_signal_matrix``), the frame-wise ``FramePlan``/``framewise_lp`` of
``tvlp.params``, and ``torch.autograd.Function``s replacing the reference's
tape-op registrations.  Every call runs hand-written sm_100a CUDA kernels
through the C ABI of ``include/tvlp.h`` (libtvlp_b200.so); there is no CPU
fallback.
"""
from . import data  # noqa: F401  (synthetic inputs; no native code)

__version__ = "0.1.0"

_LAZY = {
    "lp_forward_tv": "lpc", "lp_forward_ti": "lpc", "lp_backward_tv": "lpc",
    "lp_backward_ti": "lpc", "shift_coeffs": "lpc", "lagged_signal_matrix": "lpc",
    "lp_forward_tv_frames": "lpc", "lp_backward_tv_frames": "lpc",
    "set_validation": "lpc", "check_nonfinite": "lpc", "set_carry_precision": "lpc",
    "FramePlan": "params", "framewise_lp": "params", "expected_frame_count": "params",
    "LPTV": "autograd", "LPTI": "autograd", "LPFramewise": "autograd", "lp_tv": "autograd",
    "lp_ti": "autograd", "framewise": "autograd", "LPTVFrames": "autograd",
    "lp_tv_frames": "autograd", "lp_tv_fwd_bwd_host": "stream",
    "reflection_to_lpc": "params", "squash_reflection": "params",
    "ReflectionToLPC": "autograd",
    "gradcheck_error": "metrics",
}

__all__ = sorted(_LAZY) + ["data", "__version__"]


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    m = importlib.import_module(f".{mod}", __name__)
    return getattr(m, name)
