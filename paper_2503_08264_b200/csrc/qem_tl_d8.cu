// qem_tl_d8.cu -- the two-level kernels for latent dimension d = 8 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(8)
}  // namespace qem
