// qem_tl_d20.cu -- the two-level kernels for latent dimension d = 20 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(20)
}  // namespace qem
