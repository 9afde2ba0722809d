// qem_tl_d1.cu -- the two-level kernels for latent dimension d = 1 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(1)
}  // namespace qem
