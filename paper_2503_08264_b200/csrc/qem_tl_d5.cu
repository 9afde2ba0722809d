// qem_tl_d5.cu -- the two-level kernels for latent dimension d = 5 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(5)
}  // namespace qem
