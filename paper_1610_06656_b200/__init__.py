"""B200-native (sm_100a) hot path of SMP-PCA (arXiv 1610.06656).

The one-pass sketch ΠA, ΠB with fused exact column norms, the biased sample
Ω, the rescaled-JL estimates M̃ on Ω and WAltMin, behind the C ABI of
libsmp.so (include/smp.h).  See DESIGN.md.
"""
from .smp import (IN_CSR_F32, IN_DENSE_BF16, IN_DENSE_F32, PI_GAUSSIAN, PI_HADAMARD_TEST, PI_SRHT,  # noqa: F401
                  PI_RADEMACHER, SMPSketch, SmpError, lela, smp_pca)
