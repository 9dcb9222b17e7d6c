// Packed GF(2^d) batch verification of boolean multiplication logs (d <= 32).
//
// Over the boolean ring the verification ring is GR(2, d) = GF(2^d).  The
// reference keeps its elements as (n, d) arrays of 0/1 uint64 words and
// multiplies them on bit-packed words (grvec.py:96-115); this file keeps the
// level vectors packed from the start: one uint32 per element, bit k = the
// coefficient of x^k (128x fewer bytes than the (n, d) word layout at
// d = 16).  Products are carry-less shift/xor products reduced by the low
// terms of f (x^d = f_low(x) in characteristic 2).
//
// Characteristic 2 simplifies the reduction step (verify.py:215-241) without
// changing any value: every leg coefficient +-1 is 1, and the second
// inner-product operand f2 = 2 f1 - f0 equals f0, so
//     h(1) = sum_j f1x_j f1y_j,   h(2) = sum_j f0x_j f0y_j   (sums are xors)
// and the line evaluation is f0 + (f1 - f0) ze = f0 ^ (f0 ^ f1) ze.
//
//   r3_gfv_base_fold  level 0 straight from the base log (verify.py:168-179
//                     fused with the first reduction's folds): x'_i = r^i x_i
//                     is never formed, the h(1)/h(2) folds are xors of the
//                     powers r^i selected by the party's leg bit products, and
//                     the z power sums sum_i r^i z_i come from the same pass.
//   r3_gfv_line       one line evaluation (first level from the base bits and
//                     the powers, or a packed level) fused with the next
//                     level's h(1)/h(2) folds: a thread owns one output pair,
//                     i.e. four input rows, so the fold needs no second pass.
//
// Powers r^i are generated in registers (square-and-multiply once per thread,
// then one multiplication per grid stride); no power table is stored.
// Multiplications by the launch's constants (ze, r, r^2, r^3, the stride
// power) are nibble-table lookups in shared memory; fold products are
// accumulated as unreduced carry-less products and reduced once.  Fold
// partials are xor-reduced per block, xor-accumulated into a scratch word
// and unpacked into (rows, d) 0/1 words by the last block to finish.
#include <type_traits>

#include "r3_common.cuh"

namespace r3 {
namespace {

constexpr int GF_MAXC = 4;   // components per side
constexpr int GF_MAXT = 4;   // leg terms
constexpr int GF_MAXACC = 4;
constexpr int GF_THREADS = 256;

struct GfField {
  int d;
  u32 low;     // f without x^d
};

// a * b mod f over GF(2); a, b < 2^d.
template <bool WIDE>
__device__ __forceinline__ u32 gf_mul(u32 a, u32 b, const GfField& F) {
  if constexpr (!WIDE) {          // d <= 16: the product fits 31 bits
    u32 p = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) p ^= (b << k) & (0u - ((a >> k) & 1u));
    const u32 m = (1u << F.d) - 1u;
    while (p >> F.d) {
      const u32 hi = p >> F.d;
      p &= m;
      for (u32 g = F.low; g; g &= g - 1) p ^= hi << (__ffs(int(g)) - 1);
    }
    return p;
  } else {
    u64 p = 0;
    const u64 bb = b;
#pragma unroll
    for (int k = 0; k < 32; ++k) p ^= (bb << k) & (0ull - u64((a >> k) & 1u));
    const u64 m = (1ull << F.d) - 1ull;
    while (p >> F.d) {
      const u64 hi = p >> F.d;
      p &= m;
      for (u32 g = F.low; g; g &= g - 1) p ^= hi << (__ffs(int(g)) - 1);
    }
    return u32(p);
  }
}

// Carry-less product without the reduction (fold sums are reduced once:
// reduction mod f is GF(2)-linear).
template <bool WIDE>
__device__ __forceinline__ u64 gf_clmul(u32 a, u32 b) {
  if constexpr (!WIDE) {
    u32 p = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) p ^= (b << k) & (0u - ((a >> k) & 1u));
    return p;
  } else {
    u64 p = 0;
    const u64 bb = b;
#pragma unroll
    for (int k = 0; k < 32; ++k) p ^= (bb << k) & (0ull - u64((a >> k) & 1u));
    return p;
  }
}

__device__ __forceinline__ u32 gf_reduce(u64 p, const GfField& F) {
  const u64 m = (1ull << F.d) - 1ull;
  while (p >> F.d) {
    const u64 hi = p >> F.d;
    p &= m;
    for (u32 g = F.low; g; g &= g - 1) p ^= hi << (__ffs(int(g)) - 1);
  }
  return u32(p);
}

// Multiplication by a constant c through nibble tables in shared memory:
// T[k][n] = (n x^(4k)) c, so v c = xor_k T[k][nibble k of v] (d <= 32: at
// most 8 nibbles; the 16 entries of a row sit in distinct banks).
struct CTab {
  u32 t[8][16];
};

template <bool WIDE>
__device__ __forceinline__ void ctab_fill(CTab* tabs, const u32* consts, int ntab, const GfField& F) {
  for (int e = threadIdx.x; e < ntab * 128; e += blockDim.x) {
    const int q = e >> 7, k = (e >> 4) & 7, n = e & 15;
    tabs[q].t[k][n] = 4 * k < F.d ? gf_mul<WIDE>(u32(n) << (4 * k), consts[q], F) : 0u;
  }
}

__device__ __forceinline__ u32 ctab_mul(const CTab& T, u32 v, int d) {
  u32 o = T.t[0][v & 15] ^ T.t[1][(v >> 4) & 15] ^ T.t[2][(v >> 8) & 15] ^ T.t[3][(v >> 12) & 15];
  if (d > 16) o ^= T.t[4][(v >> 16) & 15] ^ T.t[5][(v >> 20) & 15] ^ T.t[6][(v >> 24) & 15] ^ T.t[7][v >> 28];
  return o;
}

// (1, d) 0/1 words -> packed element
__device__ __forceinline__ u32 pack_row(const u64* row, int d) {
  u32 v = 0;
  for (int k = 0; k < d; ++k) v |= u32(__ldg(row + k) & 1ull) << k;
  return v;
}

// r^e from the table R2[b] = r^(2^b)
template <bool WIDE>
__device__ __forceinline__ u32 gf_pow(const u32* R2, uint64_t e, const GfField& F) {
  u32 acc = 1;
  for (int b = 0; e; ++b, e >>= 1)
    if (e & 1) acc = gf_mul<WIDE>(acc, R2[b], F);
  return acc;
}

template <bool WIDE>
__device__ __forceinline__ void square_table(u32* R2, const u64* r, const GfField& F) {
  if (threadIdx.x == 0) {
    u32 v = pack_row(r, F.d);
    for (int b = 0; b < 48; ++b) {
      R2[b] = v;
      v = gf_mul<WIDE>(v, v, F);
    }
  }
  __syncthreads();
}

// Block xor-reduction of nacc accumulators into scratch[0..nacc); the last
// block to arrive unpacks scratch into out (nacc rows of d 0/1 words).
// scratch[7] counts finished blocks (zeroed by the launcher).
__device__ void finish_folds(u32 (&acc)[GF_MAXACC], int nacc, u32* scratch, u64* out, int d) {
  __shared__ u32 part[GF_MAXACC][GF_THREADS / 32];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < GF_MAXACC; ++q) {
    u32 v = acc[q];
#pragma unroll
    for (int o = 16; o; o >>= 1) v ^= __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part[q][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < nacc) {
    u32 v = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) v ^= part[threadIdx.x][w];
    if (v) atomicXor(scratch + threadIdx.x, v);
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(scratch + 7, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last) {
    __threadfence();
    for (int t = threadIdx.x; t < nacc * d; t += blockDim.x) {
      const u32 v = atomicOr(scratch + t / d, 0u);
      out[t] = (v >> (t % d)) & 1u;
    }
  }
}

struct GfvBaseArgs {
  const u64* x[GF_MAXC];
  const u64* y[GF_MAXC];
  const u64* z[2];
  int tx[GF_MAXT], ty[GF_MAXT];
  int ncomp, nterms, nz;
  int64_t N;
  const u64* r;
  u32* scratch;
  u64* folds;
  GfField F;
};

template <bool WIDE>
__global__ void __launch_bounds__(GF_THREADS)
gfv_base_kernel(const __grid_constant__ GfvBaseArgs A) {
  __shared__ u32 R2[48];
  __shared__ CTab T[4];                    // x r, x r^2, x r^3, x r^(4S)
  __shared__ u32 cs[4];
  square_table<WIDE>(R2, A.r, A.F);
  const int64_t nblk = (A.N + 3) / 4;
  const int64_t S = int64_t(gridDim.x) * blockDim.x;
  if (threadIdx.x == 0) {
    cs[0] = R2[0], cs[1] = R2[1], cs[2] = gf_mul<WIDE>(R2[0], R2[1], A.F);
    cs[3] = gf_pow<WIDE>(R2, uint64_t(4 * S), A.F);
  }
  __syncthreads();
  ctab_fill<WIDE>(T, cs, 4, A.F);
  __syncthreads();
  const int d = A.F.d;
  int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  u32 p = gf_pow<WIDE>(R2, uint64_t(4 * j), A.F);
  u32 acc[GF_MAXACC] = {0u, 0u, 0u, 0u};   // h1, h2, z_0, z_1
  for (; j < nblk; j += S) {
    const int64_t i0 = 4 * j;
    const u32 pw[4] = {p, ctab_mul(T[0], p, d), ctab_mul(T[1], p, d), ctab_mul(T[2], p, d)};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t i = i0 + a;
      if (i < A.N) {
        u32 xb[GF_MAXC], yb[GF_MAXC];
#pragma unroll
        for (int c = 0; c < GF_MAXC; ++c) {
          xb[c] = c < A.ncomp ? u32(__ldg(A.x[c] + i)) & 1u : 0u;
          yb[c] = c < A.ncomp ? u32(__ldg(A.y[c] + i)) & 1u : 0u;
        }
        u32 t = 0;
#pragma unroll
        for (int q = 0; q < GF_MAXT; ++q)
          if (q < A.nterms) t ^= xb[A.tx[q]] & yb[A.ty[q]];
        acc[a & 1 ? 0 : 1] ^= (0u - t) & pw[a];
#pragma unroll
        for (int c = 0; c < 2; ++c)
          if (c < A.nz) acc[2 + c] ^= (0u - (u32(__ldg(A.z[c] + i)) & 1u)) & pw[a];
      }
    }
    p = ctab_mul(T[3], p, d);
  }
  finish_folds(acc, 2 + A.nz, A.scratch, A.folds, d);
}

struct GfvLineArgs {
  const void* x[GF_MAXC];     // base 0/1 words (BASE) or packed uint32 rows
  const void* y[GF_MAXC];
  void* ox[GF_MAXC];          // packed uint32 rows, or (rows, d) words if unpacked
  void* oy[GF_MAXC];
  int tx[GF_MAXT], ty[GF_MAXT];
  int ncomp, nterms, unpacked;
  int64_t n_in;
  const u64* r;               // BASE only
  const u64* ze;
  u32* scratch;
  u64* folds;                 // NULL: no fold of the output level
  GfField F;
};

template <bool BASE>
__device__ __forceinline__ void load4(const void* src, int64_t i0, int64_t n, u32 (&v)[4]) {
  if constexpr (BASE) {
    const u64* s = static_cast<const u64*>(src);
#pragma unroll
    for (int a = 0; a < 4; ++a) v[a] = i0 + a < n ? u32(__ldg(s + i0 + a)) & 1u : 0u;
  } else {
    const u32* s = static_cast<const u32*>(src);
    if (i0 + 3 < n) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(s + i0));
      v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
    } else {
#pragma unroll
      for (int a = 0; a < 4; ++a) v[a] = i0 + a < n ? __ldg(s + i0 + a) : 0u;
    }
  }
}

__device__ __forceinline__ void store2(void* dst, int unpacked, int64_t row, int64_t n_out, u32 o0, u32 o1, int d) {
  if (!unpacked) {
    u32* o = static_cast<u32*>(dst);
    if (row + 1 < n_out) {
      *reinterpret_cast<uint2*>(o + row) = make_uint2(o0, o1);
    } else if (row < n_out) {
      o[row] = o0;
    }
  } else {
    u64* o = static_cast<u64*>(dst);
    for (int h = 0; h < 2; ++h) {
      if (row + h < n_out) {
        const u32 v = h ? o1 : o0;
        for (int k = 0; k < d; ++k) o[(row + h) * d + k] = (v >> k) & 1u;
      }
    }
  }
}

template <bool WIDE, bool BASE>
__global__ void __launch_bounds__(GF_THREADS)
gfv_line_kernel(const __grid_constant__ GfvLineArgs A) {
  __shared__ u32 R2[48];
  __shared__ CTab T[5];                    // x ze, x r, x r^2, x r^3, x r^(4S)
  __shared__ u32 cs[5];
  const GfField& F = A.F;
  const int d = F.d;
  if constexpr (BASE) square_table<WIDE>(R2, A.r, F);
  const int64_t n_out = (A.n_in + 1) / 2;
  const int64_t npair = (n_out + 1) / 2;       // a thread owns output rows 2j, 2j + 1
  const int64_t S = int64_t(gridDim.x) * blockDim.x;
  if (threadIdx.x == 0) {
    cs[0] = pack_row(A.ze, d);
    if constexpr (BASE) {
      cs[1] = R2[0], cs[2] = R2[1], cs[3] = gf_mul<WIDE>(R2[0], R2[1], F);
      cs[4] = gf_pow<WIDE>(R2, uint64_t(4 * S), F);
    }
  }
  __syncthreads();
  ctab_fill<WIDE>(T, cs, BASE ? 5 : 1, F);
  __syncthreads();
  const u32 zev = cs[0];
  const u32 om = zev ^ 1u;                     // 1 - ze = 1 + ze
  int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  u32 p = 0;
  if constexpr (BASE) p = gf_pow<WIDE>(R2, uint64_t(4 * j), F);
  using Acc = typename std::conditional<WIDE, u64, u32>::type;
  Acc h1 = 0, h2 = 0;                          // unreduced folds of the output level
  for (; j < npair; j += S) {
    const int64_t i0 = 4 * j;
    u32 wx[4];                                  // BASE: r^i (1 + ze) / r^i ze per input row
    if constexpr (BASE) {
      const u32 q1 = ctab_mul(T[1], p, d), q2 = ctab_mul(T[2], p, d), q3 = ctab_mul(T[3], p, d);
      wx[0] = ctab_mul(T[0], p, d) ^ p;
      wx[1] = ctab_mul(T[0], q1, d);
      wx[2] = ctab_mul(T[0], q2, d) ^ q2;
      wx[3] = ctab_mul(T[0], q3, d);
      p = ctab_mul(T[4], p, d);
    }
    u32 OX[GF_MAXC][2], OY[GF_MAXC][2];
#pragma unroll
    for (int c = 0; c < GF_MAXC; ++c) {
      if (c < A.ncomp) {
        u32 v[4];
        load4<BASE>(A.x[c], i0, A.n_in, v);
        if constexpr (BASE) {
          OX[c][0] = ((0u - v[0]) & wx[0]) ^ ((0u - v[1]) & wx[1]);
          OX[c][1] = ((0u - v[2]) & wx[2]) ^ ((0u - v[3]) & wx[3]);
        } else {
          OX[c][0] = v[0] ^ ctab_mul(T[0], v[0] ^ v[1], d);
          OX[c][1] = v[2] ^ ctab_mul(T[0], v[2] ^ v[3], d);
        }
        load4<BASE>(A.y[c], i0, A.n_in, v);
        if constexpr (BASE) {
          OY[c][0] = ((0u - v[0]) & om) ^ ((0u - v[1]) & zev);
          OY[c][1] = ((0u - v[2]) & om) ^ ((0u - v[3]) & zev);
        } else {
          OY[c][0] = v[0] ^ ctab_mul(T[0], v[0] ^ v[1], d);
          OY[c][1] = v[2] ^ ctab_mul(T[0], v[2] ^ v[3], d);
        }
        store2(A.ox[c], A.unpacked, 2 * j, n_out, OX[c][0], OX[c][1], d);
        store2(A.oy[c], A.unpacked, 2 * j, n_out, OY[c][0], OY[c][1], d);
      } else {
        OX[c][0] = OX[c][1] = OY[c][0] = OY[c][1] = 0u;
      }
    }
    if (A.folds) {
#pragma unroll
      for (int q = 0; q < GF_MAXT; ++q) {
        if (q < A.nterms) {
          h1 ^= Acc(gf_clmul<WIDE>(OX[A.tx[q]][1], OY[A.ty[q]][1]));
          h2 ^= Acc(gf_clmul<WIDE>(OX[A.tx[q]][0], OY[A.ty[q]][0]));
        }
      }
    }
  }
  if (A.folds) {
    u32 acc[GF_MAXACC] = {gf_reduce(h1, F), gf_reduce(h2, F), 0u, 0u};
    finish_folds(acc, 2, A.scratch, A.folds, d);
  }
}

bool valid_terms(int ncomp, int nterms, const int* tx, const int* ty) {
  if (ncomp < 1 || ncomp > GF_MAXC || nterms < 0 || nterms > GF_MAXT || (nterms && (!tx || !ty))) return false;
  for (int q = 0; q < nterms; ++q)
    if (tx[q] < 0 || tx[q] >= ncomp || ty[q] < 0 || ty[q] >= ncomp) return false;
  return true;
}

bool valid_field(int d, uint32_t f_low) {
  return d >= 1 && d <= 32 && (d == 32 || (f_low >> d) == 0) && (f_low & 1u);
}

unsigned gf_grid(int64_t work) {
  int64_t b = (work + GF_THREADS - 1) / GF_THREADS;
  const int64_t cap = int64_t(num_sms()) * 8;
  return unsigned(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace
}  // namespace r3

using namespace r3;

extern "C" int r3_gfv_base_fold(int ncomp, const uint64_t* const* x, const uint64_t* const* y, int nterms,
                                const int* tx, const int* ty, int nz, const uint64_t* const* z, int64_t N,
                                const uint64_t* r, int d, uint32_t f_low, uint64_t* folds, uint32_t* scratch,
                                void* stream) {
  if (!valid_terms(ncomp, nterms, tx, ty) || nz < 0 || nz > 2 || N < 0 || !valid_field(d, f_low) || !r ||
      !folds || !scratch || !x || !y || (nz && !z)) {
    set_error("r3_gfv_base_fold: bad arguments (ncomp %d, nterms %d, nz %d, d %d)", ncomp, nterms, nz, d);
    return R3_ERR_ARG;
  }
  GfvBaseArgs A{};
  for (int c = 0; c < ncomp; ++c) {
    A.x[c] = reinterpret_cast<const u64*>(x[c]);
    A.y[c] = reinterpret_cast<const u64*>(y[c]);
  }
  for (int c = 0; c < nz; ++c) A.z[c] = reinterpret_cast<const u64*>(z[c]);
  for (int q = 0; q < nterms; ++q) A.tx[q] = tx[q], A.ty[q] = ty[q];
  A.ncomp = ncomp, A.nterms = nterms, A.nz = nz, A.N = N;
  A.r = reinterpret_cast<const u64*>(r);
  A.scratch = scratch;
  A.folds = reinterpret_cast<u64*>(folds);
  A.F = GfField{d, f_low};
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(scratch, 0, 8 * sizeof(uint32_t), s);
  if (e != cudaSuccess) {
    set_error("r3_gfv_base_fold: memset: %s", cudaGetErrorString(e));
    return R3_ERR_CUDA;
  }
  const unsigned grid = gf_grid((N + 3) / 4);
  if (d <= 16)
    gfv_base_kernel<false><<<grid, GF_THREADS, 0, s>>>(A);
  else
    gfv_base_kernel<true><<<grid, GF_THREADS, 0, s>>>(A);
  return check_launch("r3_gfv_base_fold");
}

extern "C" int r3_gfv_line(int src_base, int ncomp, const void* const* x, const void* const* y, int64_t n_in,
                           const uint64_t* r, const uint64_t* ze, int d, uint32_t f_low, int unpacked,
                           void* const* ox, void* const* oy, int nterms, const int* tx, const int* ty,
                           uint64_t* folds, uint32_t* scratch, void* stream) {
  if (!valid_terms(ncomp, folds ? nterms : 0, tx, ty) || n_in < 0 || !valid_field(d, f_low) || !ze ||
      (src_base && !r) || !x || !y || !ox || !oy || (folds && !scratch)) {
    set_error("r3_gfv_line: bad arguments (ncomp %d, nterms %d, d %d)", ncomp, nterms, d);
    return R3_ERR_ARG;
  }
  GfvLineArgs A{};
  for (int c = 0; c < ncomp; ++c) {
    A.x[c] = x[c], A.y[c] = y[c], A.ox[c] = ox[c], A.oy[c] = oy[c];
    if (!src_base && ((reinterpret_cast<uintptr_t>(x[c]) | reinterpret_cast<uintptr_t>(y[c])) & 15)) {
      set_error("r3_gfv_line: packed inputs must be 16-byte aligned");
      return R3_ERR_ARG;
    }
    if (!unpacked && ((reinterpret_cast<uintptr_t>(ox[c]) | reinterpret_cast<uintptr_t>(oy[c])) & 7)) {
      set_error("r3_gfv_line: packed outputs must be 8-byte aligned");
      return R3_ERR_ARG;
    }
  }
  A.ncomp = ncomp, A.nterms = folds ? nterms : 0, A.unpacked = unpacked ? 1 : 0, A.n_in = n_in;
  for (int q = 0; q < A.nterms; ++q) A.tx[q] = tx[q], A.ty[q] = ty[q];
  A.r = reinterpret_cast<const u64*>(r);
  A.ze = reinterpret_cast<const u64*>(ze);
  A.scratch = scratch;
  A.folds = reinterpret_cast<u64*>(folds);
  A.F = GfField{d, f_low};
  cudaStream_t s = as_stream(stream);
  if (folds) {
    cudaError_t e = cudaMemsetAsync(scratch, 0, 8 * sizeof(uint32_t), s);
    if (e != cudaSuccess) {
      set_error("r3_gfv_line: memset: %s", cudaGetErrorString(e));
      return R3_ERR_CUDA;
    }
  }
  const int64_t n_out = (n_in + 1) / 2;
  const unsigned grid = gf_grid((n_out + 1) / 2);
  const bool wide = d > 16;
  if (src_base)
    wide ? gfv_line_kernel<true, true><<<grid, GF_THREADS, 0, s>>>(A)
         : gfv_line_kernel<false, true><<<grid, GF_THREADS, 0, s>>>(A);
  else
    wide ? gfv_line_kernel<true, false><<<grid, GF_THREADS, 0, s>>>(A)
         : gfv_line_kernel<false, false><<<grid, GF_THREADS, 0, s>>>(A);
  return check_launch("r3_gfv_line");
}
