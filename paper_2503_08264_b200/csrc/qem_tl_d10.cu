// qem_tl_d10.cu -- the two-level kernels for latent dimension d = 10 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(10)
}  // namespace qem
