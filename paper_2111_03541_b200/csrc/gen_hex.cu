// gen_hex.cu — instantiations of the element-batch kernel for ET_HEX order 1.
#include "assemble_generic.cuh"

namespace fem {

int gen_dispatch_hex(int kh, int q, const GenParams& P, cudaStream_t s, bool facet) {
  if (kh == 1) return facet ? run_q<ET_HEX, 1, 1, true>(q, P, s) : run_q<ET_HEX, 1, 1, false>(q, P, s);
  if (kh == 3) return facet ? run_q<ET_HEX, 1, 3, true>(q, P, s) : run_q<ET_HEX, 1, 3, false>(q, P, s);
  if (kh == 4) return facet ? run_q<ET_HEX, 1, 4, true>(q, P, s) : run_q<ET_HEX, 1, 4, false>(q, P, s);
  set_error("unsupported physics for this element");
  return FEM_E_UNSUPPORTED;
}

}  // namespace fem
