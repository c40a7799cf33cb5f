"""B200-native ALS-HOSVD hot path (arXiv 2004.02583) behind tenkit's API.

The product is libtenkit_b200.so (CUDA sm_100a kernels + C++ engine behind
the C-ABI in include/tenkit_b200.h); this package is its Python binding.
"""
from .tenkit import (AlsConfig, AlsReport, Context, DecompositionReport, DegenerateInitError,
                     DeviceError, DeviceTensor, HooiConfig, HooiResult, DimensionMismatchError, Error, FactorEngine,
                     FormatError, InvalidModeError, IoError, ModeOrder, ModeReport,
                     NoConvergenceError, RankTooLargeError, SingularGramError, Truncation,
                     TuckerTensor, UnsupportedError, ZeroReferenceError, als_init, als_low_rank, als_sweep,
                     default_context, frobenius_norm, gram, hooi, mode_gram, mode_n_product, multi_mode_product,
                     reconstruct, recover_singular_vectors,
                     reduced_qr, sym_eig,
                     relative_error, select_order, st_hosvd, synth_tucker, synth_tucker_slab, t_hosvd, unfold_t_times,
                     unfold_times)

__all__ = [n for n in dir() if not n.startswith("_")]
