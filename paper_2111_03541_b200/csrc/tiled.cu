// tiled.cu — node-tile owner-gather assembly (FEM_SCATTER_TILED).  Placeholder until implemented.
#include "fem_internal.cuh"

extern "C" int fem_tiles_build(fem_mesh_s* m, const int32_t* conn, int n_bsets, const int64_t* bset_len,
                               const int32_t* const* bset_elem, cudaStream_t s) {
  (void)m; (void)conn; (void)n_bsets; (void)bset_len; (void)bset_elem; (void)s;
  return 0;
}

namespace fem {
int launch_tiled(const fem_mesh_s*, const fem_pattern_s*, const fem_problem*, const double*, double*, double*,
                 cudaStream_t) {
  set_error("FEM_SCATTER_TILED not built yet");
  return FEM_E_UNSUPPORTED;
}
}  // namespace fem
