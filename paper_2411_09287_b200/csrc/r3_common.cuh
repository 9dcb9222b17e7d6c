// Shared helpers for the ring3pc B200 kernels (sm_100a).
//
// All ring values are uint64 words holding elements of Z_2^ell (ell <= 64);
// arithmetic is done mod 2^64 and results are masked to ell bits on store,
// which is exact because x -> x mod 2^ell is a ring homomorphism
// (reference grvec.py:1-7 keeps the same invariant with numpy uint64).
#pragma once

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <cuda_runtime.h>

#include "../../include/r3b200.h"

namespace r3 {

using u64 = unsigned long long;
using u32 = unsigned int;

// SM count of the current device (148 on B200), queried once per device;
// persistent grids and wave sizing use it.
int num_sms();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) once per kernel
// and device (the attribute is per device, and one process may drive
// several GPUs or launch from several threads).  False if the attribute
// could not be set.
bool smem_attr_once(const void* func, int bytes);
template <class F>
inline bool ensure_smem(F* func, int bytes) {
  return smem_attr_once(reinterpret_cast<const void*>(func), bytes);
}

// Thread-local last-error text for r3_last_error().
void set_error(const char* fmt, ...);

// Number of kernels this library has launched (every launch site goes
// through check_launch exactly once); read by r3_launch_count().
void count_launch();

inline int check_launch(const char* what) {
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return R3_ERR_CUDA;
  }
  return R3_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline unsigned grid_for(int64_t work, int threads, int max_blocks_per_sm = 8) {
  int64_t b = (work + threads - 1) / threads;
  int64_t cap = int64_t(num_sms()) * max_blocks_per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return unsigned(b);
}

// acc + a*b mod 2^64.  The compiler lowers this to IMAD.WIDE.U32 + 2 IMAD.
__device__ __forceinline__ u64 mac(u64 acc, u64 a, u64 b) { return acc + a * b; }

// Linear combination operand: row i of the operand is sum_q coef[q] * P_q[i],
// each P_q a row-strided view (stride in u64 words between rows; coefficient
// index contiguous).  Rows at or beyond nvalid[q] read as zero (this is how
// the reference's zero-lane padding of odd-length vectors is expressed,
// verify.py:220-222, without materialising a padded copy).
struct LinOperand {
  const u64* p[4];
  int64_t rowstride[4];
  int64_t nvalid[4];
  u64 coef[4];
  int nterms;
};

__device__ __forceinline__ u64 lin_load(const LinOperand& op, int64_t row, int col) {
  u64 v = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q < op.nterms && row < op.nvalid[q]) {
      v += op.coef[q] * __ldg(op.p[q] + row * op.rowstride[q] + col);
    }
  }
  return v;
}

}  // namespace r3
