"""B200-native multipoint Kronecker substitution (Harvey, arXiv 0712.4046).

Drop-in for the multiply path of the reference package ``kronmul``: the same
public names for the KS variants over Z[x] and the bivariate reductions over
Z, computed by hand-written sm_100a kernels in libkmx.so (C ABI:
include/kmx.h).  Variant names follow the reference (ksint.py:8-12):
ks2 = reciprocal (2^N, 2^-N), ks3 = negated (+-2^N).
"""
from ._lib import ReconstructionError
from .batch import BksBatch, BksModBatch, KsBatch, bks_mul_host, imad_peak, ks_mul_host, mul_engine, tc_peak
from .bipoly import (BiPoly, MissingHalveError, RingOps, bks_four, bks_negated, bks_reciprocal,
                     bks_standard, ring_z, ring_zmod)
from .modpoly import (DEFAULT_THRESHOLDS, GPU_THRESHOLDS, AutoThresholds, ModMulBatch, ModPoly, Variant,
                      choose_variant, mod_mul, mod_mul_host)
from .ksint import (derive_params, ks1_mul, ks2_mul, ks3_mul, ks4_mul, reconstruct_overlapped)
from .kstypes import (DEFAULT_MUL_CONFIG, CoeffVec, KsParams, MulConfig, MulStats, OverlapDigits)
# kronmul.pack's evaluation functions (pack.py:79-110), computed by K1; as in
# the reference, the package attribute `pack` is the function
from .pack import pack, pack_batch, pack_negated, pack_negated_reversed, pack_reversed  # noqa: E402

__version__ = "0.1.0"

__all__ = [
    "CoeffVec", "KsParams", "OverlapDigits", "MulStats", "MulConfig", "DEFAULT_MUL_CONFIG",
    "ReconstructionError", "derive_params", "ks1_mul", "ks2_mul", "ks3_mul", "ks4_mul",
    "reconstruct_overlapped", "BiPoly", "RingOps", "MissingHalveError", "ring_z", "ring_zmod",
    "bks_standard", "bks_reciprocal", "bks_negated", "bks_four", "KsBatch", "BksBatch", "BksModBatch",
    "ks_mul_host", "bks_mul_host", "imad_peak", "tc_peak", "mul_engine", "__version__",
    "ModPoly", "Variant", "AutoThresholds", "DEFAULT_THRESHOLDS", "GPU_THRESHOLDS", "choose_variant",
    "mod_mul", "ModMulBatch", "mod_mul_host",
    "pack", "pack_reversed", "pack_negated", "pack_negated_reversed", "pack_batch",
]
