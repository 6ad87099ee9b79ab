// fem_internal.cuh — library-internal structures shared by the host driver and the kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/libfem.h"
#include "physics.cuh"

namespace fem {

void set_error(const std::string& msg);

#define FEM_CUDA_TRY(call)                                                                   \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      ::fem::set_error(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " +       \
                       __FILE__ + ":" + std::to_string(__LINE__) + ": " #call);              \
      return e_ == cudaErrorMemoryAllocation ? FEM_E_OOM : FEM_E_CUDA;                       \
    }                                                                                        \
  } while (0)

// A list of assembly tasks: elements (domain terms) or (element, facet) pairs (boundary terms),
// grouped by colour: tasks [col_off[c], col_off[c+1]) share no control point.
struct TaskList {
  int64_t n = 0;
  int32_t* elem = nullptr;  // device
  int8_t* facet = nullptr;  // device (boundary sets only)
  std::vector<int64_t> col_off;  // host, size n_colours+1
};

// Node-tile schedule (FEM_SCATTER_TILED): owned points split into tiles; for tile t the elements
// touching it are tile_elem[tile_eoff[t] .. tile_eoff[t+1]).
struct TileSchedule {
  int64_t n_tiles = 0;
  int max_tile_nodes = 0;
  int64_t* tile_noff = nullptr;  // device [n_tiles+1] offsets into tile_node
  int32_t* tile_node = nullptr;  // device: owned points of each tile (ascending)
  int64_t* tile_eoff = nullptr;  // device [n_tiles+1]
  int32_t* tile_elem = nullptr;  // device: elements touching each tile
  int64_t* tile_foff = nullptr;  // device [n_bsets][n_tiles+1] facet offsets per set
  int32_t* tile_fent = nullptr;  // device: facet-entry indices (into the set's arrays) per tile
  int64_t max_tile_elems = 0;
};

}  // namespace fem

struct fem_mesh_s {
  int dim = 0, etype = 0, order = 0, physics = 0, n_loc = 0, kh = 0;
  int64_t N = 0, E = 0, own_lo = 0, own_hi = 0, n_own = 0;
  double* coords = nullptr;  // device [dim][N]
  int32_t* conn = nullptr;   // device [n_loc][E]
  fem::TaskList dom;         // element tasks, coloured
  std::vector<fem::TaskList> bnd;  // boundary set tasks, coloured
  std::vector<int64_t> bset_len;
  std::vector<int32_t*> bset_elem_dev;  // original order (device)
  std::vector<int8_t*> bset_facet_dev;
  fem::TileSchedule tiles;
  long long* err = nullptr;     // device error word: an offending element id or -1
  double* scratch_state = nullptr;  // e2e staging buffer (lazily allocated)
  size_t scratch_state_bytes = 0;
  int n_colours = 0;
};

struct fem_pattern_s {
  fem_mesh_s* mesh = nullptr;
  int64_t n_rows = 0, nnz = 0, nnz_s = 0;
  int64_t* rowptr_s = nullptr;  // device [n_own+1]
  int32_t* colidx_s = nullptr;  // device [nnz_s]
  int32_t* slot = nullptr;      // device [n_loc²][E]
  int64_t* rowptr = nullptr;    // device [n_rows+1]
  int32_t* colidx = nullptr;    // device [nnz]
};

namespace fem {

// Arguments of one assembly launch.
struct AsmArgs {
  const fem_mesh_s* m;
  const fem_pattern_s* pat;  // may be null for residual-only
  FormArgs F;
  int quad_order;
  const double* state;
  double* values;  // null: no matrix
  double* rhs;     // null: no residual
  int plain;       // 1: plain RMW (coloured), 0: atomics
  const int32_t* task_elem;  // null: identity 0..n-1
  const int8_t* task_facet;  // null for domain terms
  int64_t task_begin, task_count;
  cudaStream_t stream;
};

int launch_generic(const AsmArgs& A, bool facet);
int launch_tiled(const fem_mesh_s* m, const fem_pattern_s* pat, const fem_problem* prob,
                 const double* state, double* values, double* rhs, cudaStream_t stream);
int pattern_build(fem_mesh_s* m, cudaStream_t stream, fem_pattern_s* p);
int residual_norms(const fem_mesh_s* m, const double* rhs, double* norms, cudaStream_t stream);
FormArgs make_form_args(const fem_problem* prob, const fem_term& t);

}  // namespace fem
