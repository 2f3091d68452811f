"""Every kernel-selection path of the CUDA pipeline is parity-tested, not
only the one the shape heuristics pick: tools/paths_check.py runs in a
subprocess per forced setting (the library reads its KMX_* switches once per
process) and compares golden + BASELINE-shaped cases bit-exactly with the
oracle."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SETTINGS = [
    {"KMX_FINISH_WARP": "1"},   # warp-per-stream finish everywhere (incl. c4 long streams)
    {"KMX_FINISH_WARP": "0", "KMX_PACK_PAIR": "0"},   # block finish; one pack block per operand
    {"KMX_FINREC": "1"},        # finish + reconstruction fused (k_finrec)
    {"KMX_FINISH_CHUNKS": "1"},  # chunk-parallel finish (k_finmap + k_finchunk) everywhere
    {"KMX_FINISH_CHUNKS": "0", "KMX_SPLIT": "1"},  # warp-per-stream finish; every batch split over two streams
    {"KMX_TC": "0"},            # integer-pipe multiply everywhere
    {"KMX_TC": "1"},            # tensor-core multiply wherever supported (incl. tiny operands): swizzled-window kernel
    {"KMX_TC": "1", "KMX_FUSE_FIN": "1"},  # K2 + K3 fused in pair CTAs wherever the products are single tiles
    {"KMX_TC": "1", "KMX_TCS": "0"},  # the tiled tensor-core kernel (k_tcmul) wherever supported
    {"KMX_TC": "1", "KMX_TCS": "32"},  # swizzled-window kernel, pitch 32 (N = 32), one-shot CTAs
    {"KMX_TC": "1", "KMX_TCS": "128", "KMX_TCS_KS": "24"},  # pitch 128, many short K-chunks per tile
    {"KMX_TC": "1", "KMX_TCS": "64", "KMX_TCS_PERSIST": "1"},  # persistent warp-specialized form, pitch 64
    {"KMX_TC": "1", "KMX_TCS": "128", "KMX_TCS_PERSIST": "1", "KMX_TCS_KS": "40", "KMX_TCS_NS": "2"},  # persistent, pitch 128, short chunks, 2 stages
    {"KMX_TC": "1", "KMX_TCS": "64", "KMX_TCS_PERSIST": "2"},  # M = 64 two-window form (k_tcswz_m64), pitch 64, wherever the product fits it
    {"KMX_TC": "1", "KMX_TCS": "32", "KMX_TCS_PERSIST": "2"},  # the same at pitch 32
    {"KMX_TC": "1", "KMX_TCS": "128", "KMX_TCS_PERSIST": "2"},  # and at pitch 128 (products of up to 80 rows of 128 bytes in one K-chunk)
    {"KMX_TC": "1", "KMX_TCJ": "1", "KMX_PACK_PAIR": "2"},  # chunked single-tile tensor-core kernel; paired packs at every batch size
    {"KMX_RECON_PAIR": "2"},    # one-CTA-per-pair reconstruction (kmx_recon2.cu) for every digit width <= 64, short streams too
    {"KMX_RECON_PAIR": "0", "KMX_RECON_BIAS_SMEM": "0", "KMX_RECON_WARP": "1"},  # k_recon_par family: signed prefix sums from L2; warp-per-stream recon
    {"KMX_BIAS_FUSED": "1"},    # ks1 / ks3 signed correction inside the finish's coefficient stores (default: streaming pass)
    {"KMX_RECON_CLUSTER": "2"},  # a cluster of 2 CTAs per reconstruction stream (kmx_reconcl.cu) for every unsigned shape
    {"KMX_RECON_CLUSTER": "8", "KMX_RECON_CL_LGV": "2"},  # clusters of 8, 4 steps per thread
    {"KMX_RECON_PAIR": "0", "KMX_RECON_CLUSTER": "0", "KMX_RECON_SPEC": "1", "KMX_RECON_MINB": "0"},  # k_recon_par only (long streams unstaged): speculative stores from round 1; uncapped registers
    {"KMX_RECON_PAIR": "0", "KMX_RECON_SPEC": "0", "KMX_PACK_FAST": "0"},  # k_recon_par: separate output walk; looped pack windows only
    {"KMX_RECON_PAIR": "0", "KMX_RECON_MINB": "6", "KMX_RECON_V": "4"},  # k_recon_par: 6-CTA register cap; 4 steps per thread
    {"KMX_KARA_MIN": "600"},    # Karatsuba levels on every product above 600 limbs (tensor-core leaves)
    {"KMX_KARA_MIN": "600", "KMX_TCS": "0"},  # the same over the tiled kernel's leaves
    {"KMX_KARA_MIN": "300", "KMX_TC": "0"},  # Karatsuba over integer-pipe leaves, up to 4 levels
    {"KMX_WIDE": "1"},          # wide-digit finish + multiword reconstruction for every unsigned shape
    {"KMX_PACK_W1": "0", "KMX_PACK_CF": "0"},  # block-per-job pack everywhere (no warp-per-job, no streaming kernel)
    {"KMX_PACK_CF": "1"},       # streaming carry-free pack (kmx_packcf.cu) for every unsigned ks1 / ks2 shape
    {"KMX_PACK_CF": "1", "KMX_PACK_CF_SIGNED": "1"},  # and for signed ones (bias lift in the kernel, prefix sums by k_prefix_cf)
    {"KMX_PACK_W1": "1"},       # warp-per-job pack for every one- and two-word shape (single and paired jobs)
    {"KMX_PACK_W1": "1", "KMX_PACK_PSPLIT": "0"},  # the same with the signed prefix sums by the forward job alone
    {"KMX_PACK_SEG": "1", "KMX_BKS_UNI": "0", "KMX_BEVAL_STAGED": "0"},  # segmented pack; bivariate: IMAD products, unstaged evaluation
    {"KMX_TC_PERSIST": "2", "KMX_TC": "1", "KMX_TCS": "0"},  # persistent form of the tiled tensor-core kernel wherever it applies
]


@pytest.mark.parametrize("env", SETTINGS, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_forced_kernel_path(env):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "paths_check.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
