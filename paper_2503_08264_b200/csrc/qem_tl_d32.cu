// qem_tl_d32.cu -- the two-level kernels for latent dimension d = 32 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(32)
}  // namespace qem
