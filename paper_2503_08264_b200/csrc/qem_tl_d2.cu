// qem_tl_d2.cu -- the two-level kernels for latent dimension d = 2 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(2)
}  // namespace qem
