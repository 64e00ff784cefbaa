"""B200-native fast convolution quadrature for Riemann-Liouville derivatives (arXiv 1901.05128).

Drop-in for the reference Python package ``fraq`` (proj/python/fraq/__init__.py): the same
``__all__`` names with the same signatures, re-exported from the compiled module ``_fraq``
(paper_1901_05128_b200/csrc/fraq_py.cpp), which runs every operator on the GPU through the C ABI
in include/fraqcu.h.  There is no CPU fallback: importing without the built extension raises.

    import paper_1901_05128_b200 as fraq
    k = fraq.build_sbd_kernel(0.4, 0.05, 20, 20, 8)
    h = fraq.SbdHistory(k, fraq.HistoryVariant.standalone, 1)
"""
from __future__ import annotations

import math as _math

try:
    from . import _fraq as _impl
except ImportError as exc:  # pragma: no cover - the product must not silently degrade
    raise ImportError(
        "paper_1901_05128_b200: the CUDA extension is not built "
        "(run `python -m paper_1901_05128_b200.build`): " + str(exc)) from exc

# reference __all__ (proj/python/fraq/__init__.py:13-41)
__all__ = [
    "BeHistory",
    "FastKernelBE",
    "FastKernelSBD",
    "HistoryVariant",
    "JacobiRule",
    "KernelConfig",
    "KernelErrorReport",
    "ProblemSpec",
    "RunResult",
    "SbdHistory",
    "Scheme",
    "StateField",
    "WeightTable",
    "be_weights",
    "build_be_kernel",
    "build_sbd_kernel",
    "compute_rates",
    "coupling_from_transition",
    "default_sbd_head",
    "gauss_jacobi",
    "initial_field",
    "jacobi_moment",
    "kernel_error_report",
    "l2_norm",
    "parse_fraction",
    "run",
    "sbd_weights",
]

# B200 additions (batched / device entry points)
EXTRA = [
    "KernelBudget",
    "MultiHistory",
    "build_be_kernel_auto",
    "build_sbd_kernel_auto",
    "build_kernels_auto_sizes",
    "context_stream",
    "diag_dmma_peak",
    "fold_kernel",
    "direct_cq",
    "direct_cq_device",
    "BenchRow",
    "ConvergenceReport",
    "ConvergenceRow",
    "ExperimentConfig",
    "format_double",
    "parse_config_text",
    "parse_fraction_list",
    "resolve_config",
    "run_convergence",
    "timing_sweep",
    "dst2d",
    "dst2d_device",
    "dst_cols_device",
    "modal_run",
    "modal_run_device",
    "diag_fp64_peak",
    "gamma_fn",
    "make_be_kernel",
    "make_sbd_kernel",
    "run_2d",
    "run_batch",
    "SOLVER_AUTO",
    "SOLVER_MODAL",
    "SOLVER_PHYSICAL",
    "synchronize",
    "BandedLU",
    "BlockSystem",
    "ClassicalStepper",
    "DiscreteLaplacian",
    "FastStepper",
    "solve_block_system",
]

globals().update({name: getattr(_impl, name) for name in __all__ + EXTRA
                  if hasattr(_impl, name)})


__all__ = __all__ + EXTRA
