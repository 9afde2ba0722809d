// qem_tl_d18.cu -- the two-level kernels for latent dimension d = 18 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(18)
}  // namespace qem
