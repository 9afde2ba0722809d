// qem_tl_d4.cu -- the two-level kernels for latent dimension d = 4 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(4)
}  // namespace qem
