// stencil_g64.cu — k_tma_g instantiations for double (see stencil_g.cuh).
#include "stencil_g.cuh"

namespace sg {

void launch_stencil_g_f64(const sg_slab_desc& d, const sg_extents& e, int fn, const double* values, size_t count,
                          const void* in, void* out, cudaStream_t stream, const PeerRows& peers) {
  launch_g<double>(d, e, fn, values, count, in, out, stream, peers);
}

}  // namespace sg
