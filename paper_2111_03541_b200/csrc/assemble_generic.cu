// assemble_generic.cu — dispatch of the element-batch kernel (see assemble_generic.cuh).
#include "assemble_generic.cuh"

namespace fem {

int launch_generic(const AsmArgs& A, bool facet) {
  const fem_mesh_s* m = A.m;
  GenParams P;
  P.F = A.F;
  P.N = m->N; P.E = m->E; P.own_lo = m->own_lo; P.own_hi = m->own_hi; P.n_own = m->n_own;
  P.nnz_s = A.pat ? A.pat->nnz_s : 0;
  P.coords = m->coords; P.conn = m->conn; P.state = A.state;
  P.nu_hat = A.F.nu_hat;
  P.task_elem = A.task_elem; P.task_facet = A.task_facet;
  P.task_begin = A.task_begin; P.task_count = A.task_count;
  P.values = A.values; P.rhs = A.rhs;
  P.slot = A.pat ? A.pat->slot : nullptr;
  P.rowptr_s = A.pat ? A.pat->rowptr_s : nullptr;
  P.plain = A.plain;
  P.err = m->err;
  P.ek = A.ek; P.er = A.er; P.ek_add = A.ek_add; P.ek_nb = A.pat ? A.pat->st_nb : 0;
  P.ek_map = A.ek_map;
  const int et = m->etype, o = m->order;
  if (et == ET_TRI && o == 1) return gen_dispatch_tri(m->kh, A.quad_order, P, A.stream, facet);
  if (et == ET_HEX && o == 1) return gen_dispatch_hex(m->kh, A.quad_order, P, A.stream, facet);
  if (et == ET_TET && o == 1) return gen_dispatch_tet1(m->kh, A.quad_order, P, A.stream, facet);
  if (et == ET_TET && o == 2) return gen_dispatch_tet2(m->kh, A.quad_order, P, A.stream, facet);
  if (et == ET_HEX && o == 2) return gen_dispatch_hex2(m->kh, A.quad_order, P, A.stream, facet);
  if (et == ET_HEXS && o == 2) return gen_dispatch_hexs2(m->kh, A.quad_order, P, A.stream, facet);
  set_error("unsupported element type/order");
  return FEM_E_UNSUPPORTED;
}

}  // namespace fem
