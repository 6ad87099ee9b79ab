// gen_tri.cu — instantiations of the element-batch kernel for ET_TRI order 1.
#include "assemble_generic.cuh"

namespace fem {

int gen_dispatch_tri(int kh, int q, const GenParams& P, cudaStream_t s, bool facet) {
  if (kh == 1) return facet ? run_q<ET_TRI, 1, 1, true>(q, P, s) : run_q<ET_TRI, 1, 1, false>(q, P, s);
  if (kh == 2) return facet ? run_q<ET_TRI, 1, 2, true>(q, P, s) : run_q<ET_TRI, 1, 2, false>(q, P, s);
  set_error("unsupported physics for this element");
  return FEM_E_UNSUPPORTED;
}

}  // namespace fem
