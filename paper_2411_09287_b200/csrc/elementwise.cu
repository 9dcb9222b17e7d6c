// Elementwise share kernels: linear ops, masking, shifts, equality counts,
// axis-0 reductions and the base-ring Pi_dot legs.
//
// Reference counterparts: grvec.vmask/vneg/vscale/arith_rshift
// (grvec.py:18-51), the AShare/MVal linear maps (sharing.py:95-230), the
// fold/leg algebra of gates.dot_finish (gates.py:92-113) and P0's cross term
// gates._pair_sum (gates.py:41-49).  Contiguous same-shape operands take a
// 128-bit vectorised path; anything else goes through a strided <=4-d index
// walk (stride 0 broadcasts, mirroring numpy broadcasting in the reference).
#include <algorithm>

#include "r3_common.cuh"

namespace r3 {

__device__ __forceinline__ u64 ew_apply(int op, u64 a, u64 b) {
  switch (op) {
    case R3_EW_ADD: return a + b;
    case R3_EW_SUB: return a - b;
    case R3_EW_MUL: return a * b;
    case R3_EW_AND: return a & b;
    case R3_EW_XOR: return a ^ b;
    case R3_EW_OR: return a | b;
    case R3_EW_RSUB: return b - a;
    default: return a;
  }
}

struct Shape4 {
  int64_t s[4];
  int64_t as[4];
  int64_t bs[4];
};

template <int OP>
__global__ void ew_vec_kernel(int64_t n, u64* __restrict__ out, const u64* __restrict__ a,
                              const u64* __restrict__ b, u64 imm, u64 mask) {
  const int64_t n2 = n >> 1;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2; i += stride) {
    ulonglong2 va = reinterpret_cast<const ulonglong2*>(a)[i];
    ulonglong2 vb = b ? reinterpret_cast<const ulonglong2*>(b)[i] : make_ulonglong2(imm, imm);
    ulonglong2 r;
    r.x = ew_apply(OP, va.x, vb.x) & mask;
    r.y = ew_apply(OP, va.y, vb.y) & mask;
    reinterpret_cast<ulonglong2*>(out)[i] = r;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    u64 bv = b ? b[n - 1] : imm;
    out[n - 1] = ew_apply(OP, a[n - 1], bv) & mask;
  }
}

__global__ void ew_strided_kernel(int op, int64_t n, Shape4 sh, u64* __restrict__ out,
                                  const u64* __restrict__ a, const u64* __restrict__ b, u64 imm,
                                  u64 mask) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    int64_t rem = i, oa = 0, ob = 0;
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      int64_t idx = rem % sh.s[k];
      rem /= sh.s[k];
      oa += idx * sh.as[k];
      ob += idx * sh.bs[k];
    }
    u64 bv = b ? b[ob] : imm;
    out[i] = ew_apply(op, a[oa], bv) & mask;
  }
}

// 2-D broadcast without index division: blockIdx.y = row (row-constant /
// column-vector operands such as the edaBits weights -2^(i+1), (ell, lanes))
__global__ void ew_2d_kernel(int op, int64_t R, int64_t L, u64* __restrict__ out, const u64* __restrict__ a,
                             int64_t as0, int64_t as1, const u64* __restrict__ b, int64_t bs0, int64_t bs1,
                             u64 imm, u64 mask) {
  for (int64_t r = blockIdx.y; r < R; r += gridDim.y) {
    const u64* ar = a + r * as0;
    const u64* br = b ? b + r * bs0 : nullptr;
    u64* orow = out + r * L;
    for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < L; l += int64_t(gridDim.x) * blockDim.x) {
      const u64 bv = br ? br[l * bs1] : imm;
      orow[l] = ew_apply(op, ar[l * as1], bv) & mask;
    }
  }
}

__global__ void ars_kernel(const u64* __restrict__ a, int64_t n, int t, int width, u64* __restrict__ out) {
  const u64 mask = width == 64 ? ~0ull : ((1ull << width) - 1);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    u64 v = a[i];
    if (t == 0) {
      out[i] = v;
      continue;
    }
    u64 sign = (v >> (width - 1)) & 1ull;
    u64 fill = ((0ull - sign) << (width - t)) & mask;
    out[i] = (v >> t) | fill;
  }
}

__global__ void bit_planes_kernel(const u64* __restrict__ a, int64_t lanes, int nbits, u64* __restrict__ out) {
  const int64_t total = lanes * nbits;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += stride) {
    int64_t j = i / lanes, l = i - j * lanes;
    out[i] = (a[l] >> j) & 1ull;
  }
}

__global__ void count_ne_kernel(const u64* __restrict__ a, const u64* __restrict__ b, int64_t n,
                                u64* __restrict__ count) {
  u64 local = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    u64 bv = b ? b[i] : 0ull;
    local += (a[i] != bv);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

// out[j] (+)= sum_i a[i*rs + j]: each block owns a (rows chunk) x (column
// tile) and reduces in registers; blocks meet in exact u64 atomics (addition
// mod 2^64 is order-free, so the result is deterministic).
__global__ void sum_axis0_kernel(const u64* __restrict__ a, int64_t n, int64_t inner, int64_t rs,
                                 u64* __restrict__ out, int64_t rows_per_block) {
  const int64_t col = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (col >= inner) return;
  const int64_t r0 = blockIdx.y * rows_per_block;
  const int64_t r1 = min(n, r0 + rows_per_block);
  u64 acc = 0;
  for (int64_t r = r0; r < r1; ++r) acc += a[r * rs + col];
  atomicAdd(out + col, acc);
}

__global__ void mask_kernel(u64* out, int64_t n, u64 mask) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) out[i] &= mask;
}

__global__ void dot_fold_kernel(int64_t n, int64_t lanes, const u64* __restrict__ a, int64_t a_rs,
                                int64_t a_ls, const u64* __restrict__ b, int64_t b_rs, int64_t b_ls,
                                u64* __restrict__ out, u64 mask) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < lanes; l += stride) {
    u64 acc = 0;
    for (int64_t i = 0; i < n; ++i) acc += a[i * a_rs + l * a_ls] * b[i * b_rs + l * b_ls];
    out[l] = acc & mask;
  }
}

template <int ROLE>
__global__ void mul_leg_kernel(int64_t n, int64_t lanes, const u64* __restrict__ mx, int64_t mx_rs,
                               int64_t mx_ls, const u64* __restrict__ my, int64_t my_rs, int64_t my_ls,
                               const u64* __restrict__ sx, int64_t sx_rs, int64_t sx_ls,
                               const u64* __restrict__ sy, int64_t sy_rs, int64_t sy_ls,
                               const u64* __restrict__ g, u64* __restrict__ out, u64 mask) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < lanes; l += stride) {
    u64 acc = g[l];
    for (int64_t i = 0; i < n; ++i) {
      u64 vmx = mx[i * mx_rs + l * mx_ls], vmy = my[i * my_rs + l * my_ls];
      u64 vsx = sx[i * sx_rs + l * sx_ls], vsy = sy[i * sy_rs + l * sy_ls];
      if (ROLE == 1) {
        acc -= vmx * vsy + vmy * vsx;
      } else {
        acc += vmx * (vmy - vsy) - vmy * vsx;
      }
    }
    out[l] = acc & mask;
  }
}

}  // namespace r3

using namespace r3;

static bool contiguous_full(int ndim, const int64_t* shape, const int64_t* st) {
  int64_t expect = 1;
  for (int k = ndim - 1; k >= 0; --k) {
    if (shape[k] != 1 && st[k] != expect) return false;
    expect *= shape[k];
  }
  return true;
}

extern "C" int r3_ew(int op, int ndim, const int64_t* shape, uint64_t* out, const uint64_t* a,
                     const int64_t* a_strides, const uint64_t* b, const int64_t* b_strides,
                     uint64_t imm, uint64_t mask, void* stream) {
  if (ndim < 0 || ndim > 4 || op < 0 || op > R3_EW_COPY || !out || !a) {
    set_error("r3_ew: bad arguments (op=%d ndim=%d)", op, ndim);
    return R3_ERR_ARG;
  }
  int64_t n = 1;
  for (int k = 0; k < ndim; ++k) n *= shape[k];
  if (n == 0) return R3_OK;
  cudaStream_t s = as_stream(stream);
  const bool ca = contiguous_full(ndim, shape, a_strides);
  const bool cb = (b == nullptr) || contiguous_full(ndim, shape, b_strides);
  const bool aligned = ((uintptr_t(out) | uintptr_t(a) | uintptr_t(b)) & 15) == 0;
  if (op == R3_EW_COPY) b = nullptr;
  if (ca && cb && aligned) {
    unsigned grid = grid_for((n + 1) / 2, 256, 8);
#define R3_EW_CASE(OPC) \
  case OPC: ew_vec_kernel<OPC><<<grid, 256, 0, s>>>(n, (u64*)out, (const u64*)a, (const u64*)b, imm, mask); break;
    switch (op) {
      R3_EW_CASE(R3_EW_ADD)
      R3_EW_CASE(R3_EW_SUB)
      R3_EW_CASE(R3_EW_MUL)
      R3_EW_CASE(R3_EW_AND)
      R3_EW_CASE(R3_EW_XOR)
      R3_EW_CASE(R3_EW_OR)
      R3_EW_CASE(R3_EW_RSUB)
      R3_EW_CASE(R3_EW_COPY)
    }
#undef R3_EW_CASE
    return check_launch("r3_ew(vec)");
  }
  // 2-D (or 2-D after dropping leading unit dims): row-wise kernel
  {
    int k0 = 0;
    while (k0 < ndim - 2 && shape[k0] == 1) ++k0;
    if (ndim - k0 == 2) {
      const int64_t R = shape[k0], L = shape[k0 + 1];
      const unsigned gy = unsigned(R < 65535 ? R : 65535);
      const int64_t want = (int64_t(num_sms()) * 8 + gy - 1) / gy;
      const unsigned gx = unsigned(std::max<int64_t>(1, std::min<int64_t>(want, (L + 255) / 256)));
      ew_2d_kernel<<<dim3(gx, gy), 256, 0, s>>>(op, R, L, (u64*)out, (const u64*)a, a_strides[k0],
                                                a_strides[k0 + 1], (const u64*)b, b ? b_strides[k0] : 0,
                                                b ? b_strides[k0 + 1] : 0, imm, mask);
      return check_launch("r3_ew(2d)");
    }
  }
  Shape4 sh;
  for (int k = 0; k < 4; ++k) {
    int src = k - (4 - ndim);
    sh.s[k] = src >= 0 ? shape[src] : 1;
    sh.as[k] = src >= 0 ? a_strides[src] : 0;
    sh.bs[k] = (src >= 0 && b) ? b_strides[src] : 0;
  }
  ew_strided_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(op, n, sh, (u64*)out, (const u64*)a,
                                                       (const u64*)b, imm, mask);
  return check_launch("r3_ew(strided)");
}

extern "C" int r3_ew_flat(int op, int64_t n, uint64_t* out, const uint64_t* a, const uint64_t* b,
                          uint64_t imm, uint64_t mask, void* stream) {
  // contiguous fast path of r3_ew (one call, no shape/stride arrays)
  const int64_t shape[1] = {n};
  const int64_t st[1] = {1};
  return r3_ew(op, 1, shape, out, a, st, b, st, imm, mask, stream);
}

// out = (a - b - c) & mask (op 0) or (a + b + c) & mask (op 1): the
// reconstruction of an opened value from the three views (sharing.rec,
// sharing.py:364-471) in one pass instead of two subtractions.
__global__ void ew3_kernel(int op, int64_t n, u64* __restrict__ out, const u64* __restrict__ a,
                           const u64* __restrict__ b, const u64* __restrict__ c, u64 mask) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    out[i] = (op == 0 ? a[i] - b[i] - c[i] : a[i] + b[i] + c[i]) & mask;
}

extern "C" int r3_ew3(int op, int64_t n, uint64_t* out, const uint64_t* a, const uint64_t* b,
                      const uint64_t* c, uint64_t mask, void* stream) {
  if ((op != 0 && op != 1) || n < 0) {
    set_error("r3_ew3: bad arguments");
    return R3_ERR_ARG;
  }
  if (n == 0) return R3_OK;
  ew3_kernel<<<grid_for(n, 256, 8), 256, 0, as_stream(stream)>>>(op, n, (u64*)out, (const u64*)a,
                                                                 (const u64*)b, (const u64*)c, mask);
  return check_launch("r3_ew3");
}

struct Ptr4 {
  const u64* p[4];
};
struct OutPtr4 {
  u64* p[4];
};

// k same-length contiguous components in one launch (blockIdx.y = component):
// the fields of one party's share view (s1, s2, total, m) move together.
template <typename T>
__device__ __forceinline__ T pick4(const T (&p)[4], int c) {
  // select without dynamic indexing (keeps the parameter arrays out of local memory)
  return c == 0 ? p[0] : c == 1 ? p[1] : c == 2 ? p[2] : p[3];
}

template <int OP>
__global__ void ew_multi_kernel(int64_t n, OutPtr4 out, Ptr4 a, Ptr4 b, u64 imm, u64 mask) {
  const int c = blockIdx.y;
  const u64* __restrict__ pa = pick4(a.p, c);
  const u64* __restrict__ pb = pick4(b.p, c);
  u64* __restrict__ po = pick4(out.p, c);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const bool vec = ((uintptr_t(pa) | uintptr_t(pb) | uintptr_t(po)) & 15) == 0;
  if (vec) {
    const int64_t n2 = n / 2;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2; i += stride) {
      const ulonglong2 x = reinterpret_cast<const ulonglong2*>(pa)[i];
      const ulonglong2 y = pb ? reinterpret_cast<const ulonglong2*>(pb)[i] : make_ulonglong2(imm, imm);
      reinterpret_cast<ulonglong2*>(po)[i] =
          make_ulonglong2(ew_apply(OP, x.x, y.x) & mask, ew_apply(OP, x.y, y.y) & mask);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
      po[n - 1] = ew_apply(OP, pa[n - 1], pb ? pb[n - 1] : imm) & mask;
    return;
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    po[i] = ew_apply(OP, pa[i], pb ? pb[i] : imm) & mask;
}

extern "C" int r3_ew_multi(int op, int k, int64_t n, uint64_t* const* out, const uint64_t* const* a,
                           const uint64_t* const* b, uint64_t imm, uint64_t mask, void* stream) {
  if (k < 1 || k > 4 || n < 0 || op < 0 || op > R3_EW_COPY) {
    set_error("r3_ew_multi: bad arguments (op=%d k=%d)", op, k);
    return R3_ERR_ARG;
  }
  if (n == 0) return R3_OK;
  OutPtr4 o{};
  Ptr4 pa{}, pb{};
  for (int c = 0; c < k; ++c) {
    o.p[c] = reinterpret_cast<u64*>(out[c]);
    pa.p[c] = reinterpret_cast<const u64*>(a[c]);
    pb.p[c] = (b && op != R3_EW_COPY) ? reinterpret_cast<const u64*>(b[c]) : nullptr;
  }
  cudaStream_t s = as_stream(stream);
  const unsigned gx = grid_for(n, 256, 8);
  const unsigned gxk = (gx + k - 1) / k;
  const dim3 grid{gxk > 0 ? gxk : 1u, unsigned(k), 1};
  switch (op) {
#define R3_EWM_CASE(OPC) \
  case OPC: ew_multi_kernel<OPC><<<grid, 256, 0, s>>>(n, o, pa, pb, imm, mask); break;
    R3_EWM_CASE(R3_EW_ADD)
    R3_EWM_CASE(R3_EW_SUB)
    R3_EWM_CASE(R3_EW_MUL)
    R3_EWM_CASE(R3_EW_AND)
    R3_EWM_CASE(R3_EW_XOR)
    R3_EWM_CASE(R3_EW_OR)
    R3_EWM_CASE(R3_EW_RSUB)
    R3_EWM_CASE(R3_EW_COPY)
#undef R3_EWM_CASE
  }
  return check_launch("r3_ew_multi");
}

extern "C" int r3_ars(const uint64_t* a, int64_t n, int t, int width, uint64_t* out, void* stream) {
  if (width < 1 || width > 64 || t < 0 || t >= width || n < 0) {
    set_error("r3_ars: shift %d out of range for width %d", t, width);
    return R3_ERR_ARG;
  }
  if (n == 0) return R3_OK;
  ars_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>((const u64*)a, n, t, width, (u64*)out);
  return check_launch("r3_ars");
}

extern "C" int r3_bit_planes(const uint64_t* a, int64_t lanes, int nbits, uint64_t* out, void* stream) {
  if (nbits < 1 || nbits > 64 || lanes < 0) {
    set_error("r3_bit_planes: bad arguments");
    return R3_ERR_ARG;
  }
  if (lanes == 0) return R3_OK;
  bit_planes_kernel<<<grid_for(lanes * nbits, 256), 256, 0, as_stream(stream)>>>((const u64*)a, lanes, nbits,
                                                                                   (u64*)out);
  return check_launch("r3_bit_planes");
}

extern "C" int r3_count_nonequal(const uint64_t* a, const uint64_t* b, int64_t n, uint64_t* count,
                                 void* stream) {
  if (n < 0 || !count) {
    set_error("r3_count_nonequal: bad arguments");
    return R3_ERR_ARG;
  }
  if (n == 0) return R3_OK;
  count_ne_kernel<<<grid_for(n, 256, 4), 256, 0, as_stream(stream)>>>((const u64*)a, (const u64*)b, n,
                                                                       (u64*)count);
  return check_launch("r3_count_nonequal");
}

extern "C" int r3_sum_axis0(const uint64_t* a, int64_t n, int64_t inner, int64_t rowstride, uint64_t* out,
                            uint64_t mask, int accumulate, void* stream) {
  if (n < 0 || inner < 0) {
    set_error("r3_sum_axis0: bad arguments");
    return R3_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  if (inner == 0) return R3_OK;
  if (!accumulate) {
    cudaError_t e = cudaMemsetAsync(out, 0, size_t(inner) * 8, s);
    if (e != cudaSuccess) {
      set_error("r3_sum_axis0: memset: %s", cudaGetErrorString(e));
      return R3_ERR_CUDA;
    }
  }
  if (n > 0) {
    const int threads = inner >= 256 ? 256 : (inner >= 64 ? 64 : 32);
    const int64_t colblocks = (inner + threads - 1) / threads;
    // aim for ~8 resident blocks per SM in total
    int64_t ychunks = (int64_t(num_sms()) * 8 + colblocks - 1) / colblocks;
    int64_t rows_per_block = (n + ychunks - 1) / ychunks;
    if (rows_per_block < 16) rows_per_block = 16;
    ychunks = (n + rows_per_block - 1) / rows_per_block;
    if (ychunks > 65535) {
      ychunks = 65535;
      rows_per_block = (n + ychunks - 1) / ychunks;
    }
    dim3 grid{unsigned(colblocks), unsigned(ychunks), 1u};
    sum_axis0_kernel<<<grid, threads, 0, s>>>((const u64*)a, n, inner, rowstride, (u64*)out, rows_per_block);
    int rc = check_launch("r3_sum_axis0");
    if (rc) return rc;
  }
  if (mask != ~0ull) {
    mask_kernel<<<grid_for(inner, 256), 256, 0, s>>>((u64*)out, inner, mask);
    return check_launch("r3_sum_axis0(mask)");
  }
  return R3_OK;
}

extern "C" int r3_dot_fold(int64_t n, int64_t lanes, const uint64_t* a, int64_t a_rs, int64_t a_ls,
                           const uint64_t* b, int64_t b_rs, int64_t b_ls, uint64_t* out, uint64_t mask,
                           void* stream) {
  if (n < 0 || lanes < 0) {
    set_error("r3_dot_fold: bad arguments");
    return R3_ERR_ARG;
  }
  if (lanes == 0) return R3_OK;
  dot_fold_kernel<<<grid_for(lanes, 256), 256, 0, as_stream(stream)>>>(n, lanes, (const u64*)a, a_rs, a_ls,
                                                                       (const u64*)b, b_rs, b_ls, (u64*)out,
                                                                       mask);
  return check_launch("r3_dot_fold");
}

extern "C" int r3_mul_leg(int role, int64_t n, int64_t lanes, const uint64_t* mx, int64_t mx_rs, int64_t mx_ls,
                          const uint64_t* my, int64_t my_rs, int64_t my_ls, const uint64_t* sx, int64_t sx_rs,
                          int64_t sx_ls, const uint64_t* sy, int64_t sy_rs, int64_t sy_ls, const uint64_t* g,
                          uint64_t* out, uint64_t mask, void* stream) {
  if ((role != 1 && role != 2) || n < 0 || lanes < 0) {
    set_error("r3_mul_leg: bad arguments (role=%d)", role);
    return R3_ERR_ARG;
  }
  if (lanes == 0) return R3_OK;
  unsigned grid = grid_for(lanes, 256);
  cudaStream_t s = as_stream(stream);
  if (role == 1)
    mul_leg_kernel<1><<<grid, 256, 0, s>>>(n, lanes, (const u64*)mx, mx_rs, mx_ls, (const u64*)my, my_rs, my_ls,
                                            (const u64*)sx, sx_rs, sx_ls, (const u64*)sy, sy_rs, sy_ls,
                                            (const u64*)g, (u64*)out, mask);
  else
    mul_leg_kernel<2><<<grid, 256, 0, s>>>(n, lanes, (const u64*)mx, mx_rs, mx_ls, (const u64*)my, my_rs, my_ls,
                                            (const u64*)sx, sx_rs, sx_ls, (const u64*)sy, sy_rs, sy_ls,
                                            (const u64*)g, (u64*)out, mask);
  return check_launch("r3_mul_leg");
}

// ---------------------------------------------------------------------------
// The local arithmetic of one verification reduction round for all three
// simulated parties (verify._round_joint; gates.py:52-177 for the two vfy.dot
// gates of single GR elements, sharing.py:364-420 for the opened even point):
//   om_tot[g] = om_s1[g] + om_s2[g]                 (P0's output-mask sum)
//   g_s2[g]   = F0[g] + om_tot[g] - g_s1[g]         (P0 -> P2: Gamma - s1)
//   leg1[g]   = F1[g] + g_s1[g],  leg2[g] = F2[g] + g_s2[g],  m[g] = leg1 + leg2
//   S1 = 2 zeta.s1, S2 = 2 zeta.s2, M = 2 zeta.m, ze = M - S1 - S2
// for the gates g = 0, 1; d01 rows = (om1.s1, g1.s1, om2.s1, g2.s1), d02 rows =
// (om1.s2, om2.s2).  out rows: om_tot[2], g_s2[2], leg1[2], leg2[2], m[2], S1,
// S2, M, ze (14 rows of d words).  One thread per coefficient.
__global__ void vfy_round_kernel(int d, const u64* __restrict__ F0, const u64* __restrict__ F1,
                                 const u64* __restrict__ F2, const u64* __restrict__ d01,
                                 const u64* __restrict__ d02, const u64* __restrict__ zs1,
                                 const u64* __restrict__ zs2, const u64* __restrict__ zm, u64* __restrict__ out,
                                 u64 mask) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= d) return;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const u64 os1 = d01[(2 * g) * d + k], gs1 = d01[(2 * g + 1) * d + k], os2 = d02[g * d + k];
    const u64 tot = os1 + os2;
    const u64 gs2 = F0[g * d + k] + tot - gs1;
    const u64 l1 = F1[g * d + k] + gs1, l2 = F2[g * d + k] + gs2;
    out[(0 + g) * d + k] = tot & mask;
    out[(2 + g) * d + k] = gs2 & mask;
    out[(4 + g) * d + k] = l1 & mask;
    out[(6 + g) * d + k] = l2 & mask;
    out[(8 + g) * d + k] = (l1 + l2) & mask;
  }
  const u64 s1 = 2 * zs1[k], s2 = 2 * zs2[k], m = 2 * zm[k];
  out[10 * d + k] = s1 & mask;
  out[11 * d + k] = s2 & mask;
  out[12 * d + k] = m & mask;
  out[13 * d + k] = (m - s1 - s2) & mask;
}

extern "C" int r3_vfy_round(int d, const uint64_t* F0, const uint64_t* F1, const uint64_t* F2, const uint64_t* d01,
                            const uint64_t* d02, const uint64_t* zs1, const uint64_t* zs2, const uint64_t* zm,
                            uint64_t* out, uint64_t mask, void* stream) {
  if (d < 1 || d > 1024 || !F0 || !F1 || !F2 || !d01 || !d02 || !zs1 || !zs2 || !zm || !out) {
    set_error("r3_vfy_round: bad arguments");
    return R3_ERR_ARG;
  }
  vfy_round_kernel<<<(d + 127) / 128, 128, 0, as_stream(stream)>>>(
      d, (const u64*)F0, (const u64*)F1, (const u64*)F2, (const u64*)d01, (const u64*)d02, (const u64*)zs1,
      (const u64*)zs2, (const u64*)zm, (u64*)out, mask);
  return check_launch("r3_vfy_round");
}

// out_c = (a_c + b_c - 2 p_c) & mask for k <= 4 same-length components
// (blockIdx.y = component): the arithmetic XOR of bit shares a ^ b =
// a + b - 2ab (nonlinear.py:43-55, edaBits / daBits) in one pass instead of
// an addition, a public scaling and a subtraction.
__global__ void xor_arith_kernel(int64_t n, OutPtr4 out, Ptr4 a, Ptr4 b, Ptr4 p, u64 mask) {
  const int c = blockIdx.y;
  const u64* __restrict__ pa = pick4(a.p, c);
  const u64* __restrict__ pb = pick4(b.p, c);
  const u64* __restrict__ pp = pick4(p.p, c);
  u64* __restrict__ po = pick4(out.p, c);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const bool vec = ((uintptr_t(pa) | uintptr_t(pb) | uintptr_t(pp) | uintptr_t(po)) & 15) == 0;
  if (vec) {
    const int64_t n2 = n / 2;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2; i += stride) {
      const ulonglong2 x = reinterpret_cast<const ulonglong2*>(pa)[i];
      const ulonglong2 y = reinterpret_cast<const ulonglong2*>(pb)[i];
      const ulonglong2 z = reinterpret_cast<const ulonglong2*>(pp)[i];
      reinterpret_cast<ulonglong2*>(po)[i] =
          make_ulonglong2((x.x + y.x - 2 * z.x) & mask, (x.y + y.y - 2 * z.y) & mask);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) po[n - 1] = (pa[n - 1] + pb[n - 1] - 2 * pp[n - 1]) & mask;
    return;
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    po[i] = (pa[i] + pb[i] - 2 * pp[i]) & mask;
}

extern "C" int r3_xor_arith(int k, int64_t n, uint64_t* const* out, const uint64_t* const* a,
                            const uint64_t* const* b, const uint64_t* const* p, uint64_t mask, void* stream) {
  if (k < 1 || k > 4 || n < 0 || !out || !a || !b || !p) {
    set_error("r3_xor_arith: bad arguments (1 <= k <= 4)");
    return R3_ERR_ARG;
  }
  if (n == 0) return R3_OK;
  OutPtr4 o{};
  Ptr4 pa{}, pb{}, pp{};
  for (int c = 0; c < k; ++c) {
    if (!out[c] || !a[c] || !b[c] || !p[c]) {
      set_error("r3_xor_arith: null component");
      return R3_ERR_ARG;
    }
    o.p[c] = reinterpret_cast<u64*>(out[c]);
    pa.p[c] = reinterpret_cast<const u64*>(a[c]);
    pb.p[c] = reinterpret_cast<const u64*>(b[c]);
    pp.p[c] = reinterpret_cast<const u64*>(p[c]);
  }
  const dim3 grid(grid_for((n + 1) / 2, 256, 8), unsigned(k));
  xor_arith_kernel<<<grid, 256, 0, as_stream(stream)>>>(n, o, pa, pb, pp, mask);
  return check_launch("r3_xor_arith");
}

// out_c[l] = sum_{i < rows} w[i] (a_c[i L + l] + b_c[i L + l]) & mask for k <= 4
// components of (rows, L) arrays: the linear part of the edaBits
// recomposition, sum_i 2^i (m_i + r'_i) (nonlinear.py:104-118), without
// writing the (rows, L) scaled sum.  One thread per lane (coalesced rows).
__global__ void wsum_rows_kernel(int rows, int64_t L, OutPtr4 out, Ptr4 a, Ptr4 b, const u64* __restrict__ w,
                                 u64 mask) {
  const int c = blockIdx.y;
  const u64* __restrict__ pa = pick4(a.p, c);
  const u64* __restrict__ pb = pick4(b.p, c);
  u64* __restrict__ po = pick4(out.p, c);
  __shared__ u64 sw[64];
  for (int i = threadIdx.x; i < rows && i < 64; i += blockDim.x) sw[i] = w[i];
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < L; l += stride) {
    u64 acc = 0;
#pragma unroll 8
    for (int i = 0; i < rows; ++i) acc += sw[i] * (__ldg(pa + i * L + l) + __ldg(pb + i * L + l));
    po[l] = acc & mask;
  }
}

extern "C" int r3_wsum_rows(int k, int rows, int64_t L, uint64_t* const* out, const uint64_t* const* a,
                            const uint64_t* const* b, const uint64_t* w, uint64_t mask, void* stream) {
  if (k < 1 || k > 4 || rows < 1 || rows > 64 || L < 0 || !out || !a || !b || !w) {
    set_error("r3_wsum_rows: bad arguments (1 <= k <= 4, 1 <= rows <= 64)");
    return R3_ERR_ARG;
  }
  if (L == 0) return R3_OK;
  OutPtr4 o{};
  Ptr4 pa{}, pb{};
  for (int c = 0; c < k; ++c) {
    if (!out[c] || !a[c] || !b[c]) {
      set_error("r3_wsum_rows: null component");
      return R3_ERR_ARG;
    }
    o.p[c] = reinterpret_cast<u64*>(out[c]);
    pa.p[c] = reinterpret_cast<const u64*>(a[c]);
    pb.p[c] = reinterpret_cast<const u64*>(b[c]);
  }
  const dim3 grid(grid_for(L, 256, 8), unsigned(k));
  wsum_rows_kernel<<<grid, 256, 0, as_stream(stream)>>>(rows, L, o, pa, pb, (const u64*)w, mask);
  return check_launch("r3_wsum_rows");
}

// out_c[i L + l] = w[i] a_c[i L + l] & mask for k <= 4 components of (rows, L)
// arrays (a public per-row scaling, e.g. the -2^(i+1) x side of the edaBits
// inner product, nonlinear.py:104-118): 128-bit accesses, one launch for
// every field instead of one broadcasting launch per field.
__global__ void scale_rows_kernel(int rows, int64_t L, OutPtr4 out, Ptr4 a, const u64* __restrict__ w, u64 mask) {
  const int c = blockIdx.y;
  const u64* __restrict__ pa = pick4(a.p, c);
  u64* __restrict__ po = pick4(out.p, c);
  const int64_t n = int64_t(rows) * L;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const bool vec = ((uintptr_t(pa) | uintptr_t(po)) & 15) == 0 && (L & 1) == 0;
  if (vec) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n / 2; i += stride) {
      const u64 s = __ldg(w + (2 * i) / L);
      const ulonglong2 x = reinterpret_cast<const ulonglong2*>(pa)[i];
      reinterpret_cast<ulonglong2*>(po)[i] = make_ulonglong2((s * x.x) & mask, (s * x.y) & mask);
    }
    return;
  }
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    po[i] = (__ldg(w + i / L) * pa[i]) & mask;
}

extern "C" int r3_scale_rows(int k, int rows, int64_t L, uint64_t* const* out, const uint64_t* const* a,
                             const uint64_t* w, uint64_t mask, void* stream) {
  if (k < 1 || k > 4 || rows < 1 || L < 0 || !out || !a || !w) {
    set_error("r3_scale_rows: bad arguments (1 <= k <= 4)");
    return R3_ERR_ARG;
  }
  if (L == 0) return R3_OK;
  OutPtr4 o{};
  Ptr4 pa{};
  for (int c = 0; c < k; ++c) {
    if (!out[c] || !a[c]) {
      set_error("r3_scale_rows: null component");
      return R3_ERR_ARG;
    }
    o.p[c] = reinterpret_cast<u64*>(out[c]);
    pa.p[c] = reinterpret_cast<const u64*>(a[c]);
  }
  const dim3 grid(grid_for((int64_t(rows) * L + 1) / 2, 256, 8), unsigned(k));
  scale_rows_kernel<<<grid, 256, 0, as_stream(stream)>>>(rows, L, o, pa, (const u64*)w, mask);
  return check_launch("r3_scale_rows");
}
