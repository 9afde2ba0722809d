// qem_tl_d7.cu -- the two-level kernels for latent dimension d = 7 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(7)
}  // namespace qem
