// Internal (C++) interfaces between the CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/leanot_b200.h"
#include "leanot_common.cuh"

namespace leanot {

struct RowPassArgs {
  CostView cost;
  int64_t i0, i1;              // global rows [i0, i1)
  const double* a;             // K device scalars
  const double* b[LEANOT_MAX_K];
  const int64_t* shift;        // shift[(k / shift_kgroup) * shift_kstride + (i-i0)] (shift_at)
  int64_t shift_kstride;       // 0: one shift per row shared by all weight sets
  int shift_kgroup;            // weight sets per shift group (0 or 1: every set its own stride)
  double* S;                   // K x nr row sums
  int64_t* m_used;             // K x nr shifts used (may be null)
  // evaluation sweep (weight set 0)
  double* rowstat;             // 3 x nr: sum e*C, sum e*x, min_j (C_ij + sd_j)
  const double* sd;
  // finalize: column-pass coefficients g*EC{0..3}, g = rw_i / S (rw null: g = 1/S)
  const double* rw;            // indexed by global row
  double* coef;                // K x nr x 4 (may be null)
  int64_t* shift_next;         // nr (may be null)
  int next_from_k;
  int next_group;              // > 0: sets k with k % next_group == next_from_k write
                               // shift_next[(k / next_group) * nr + li] (batched barycenter marginals)
  int32_t* flags;              // [count, -, (k, li)...]
  int gram;                    // 1: points p = 2 with norms -> expanded-form sweep (CostGram)
};

struct ColPassArgs {
  CostView cost;
  int64_t i0, i1;
  const double* a;
  const double* b[LEANOT_MAX_K];
  const int64_t* m;            // K x nr
  const double* coef;          // K x nr x 4
  double* slab;                // splits x K x n
  int splits;
  int gram;                    // must match the pass A that produced m / coef
};

// row shift of weight set k, local row li
__host__ __device__ inline int64_t shift_at(const RowPassArgs& A, int k, int64_t li) {
  const int g = A.shift_kgroup > 1 ? k / A.shift_kgroup : k;
  return A.shift[g * A.shift_kstride + li];
}

int num_sms();
bool gram_enabled();
int launch_rowpass(const RowPassArgs& A, int K, bool eval, cudaStream_t st);
int launch_rowmax(const RowPassArgs& A, int K, int64_t* out, cudaStream_t st);
int launch_colpass(const ColPassArgs& A, int K, cudaStream_t st);
int launch_slab_reduce(const double* slab, int splits, int K, int64_t n, double* col, cudaStream_t st);
// vmin (optional, scale < 0, sgn = 1): per-row min_j (C_ij + v_j) from pass A -> exact shift, one read
int launch_rowlse(const CostView& cv, int64_t i0, int64_t i1, const double* v, double sgn, double scale, double* L,
                  cudaStream_t st, const double* vmin = nullptr);
int launch_rowmin(const CostView& cv, int64_t i0, int64_t i1, const double* v, double* out, cudaStream_t st);
int launch_cost_block(const CostView& cv, int64_t i0, int64_t i1, double* out, int64_t ldo, cudaStream_t st);

void set_error(const char* fmt, ...);
int check_launch(const char* what);

}  // namespace leanot
