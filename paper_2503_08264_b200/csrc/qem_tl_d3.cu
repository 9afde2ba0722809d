// qem_tl_d3.cu -- the two-level kernels for latent dimension d = 3 (qem_two_level.cuh).
#include "qem_two_level.cuh"

namespace qem {
QEM_TL_INSTANTIATE(3)
}  // namespace qem
