// gen_tet2.cu — instantiations of the element-batch kernel for ET_TET order 2.
#include "assemble_generic.cuh"

namespace fem {

int gen_dispatch_tet2(int kh, int q, const GenParams& P, cudaStream_t s, bool facet) {
  if (kh == 1) return facet ? run_q<ET_TET, 2, 1, true>(q, P, s) : run_q<ET_TET, 2, 1, false>(q, P, s);
  if (kh == 3) return facet ? run_q<ET_TET, 2, 3, true>(q, P, s) : run_q<ET_TET, 2, 3, false>(q, P, s);
  if (kh == 4) return facet ? run_q<ET_TET, 2, 4, true>(q, P, s) : run_q<ET_TET, 2, 4, false>(q, P, s);
  set_error("unsupported physics for this element");
  return FEM_E_UNSUPPORTED;
}

}  // namespace fem
