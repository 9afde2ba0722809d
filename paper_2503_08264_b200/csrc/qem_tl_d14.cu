// qem_tl_d14.cu -- the two-level kernels for latent dimension d = 14 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(14)
}  // namespace qem
