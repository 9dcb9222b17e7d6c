// Galois-ring GR(2^ell, d) kernels and the fused verification stages.
//
// Reference counterparts: grvec.gr_mul / gr_dot / gr_powers / gr_line_eval
// (grvec.py:78-167), the fixed sparse moduli f = x^d + g(x) of rings.py:180-188
// and the compress / reduce stages of verify.py:126-241.
//
// Reduction mod f without the reference's dense (d-1, d) reduction matrix:
// with x^d = -g (deg g <= 7 for every supported d), a product
// p = low + x^d * high reduces as  low - t_low + g * t_high  where
// t = g * high = t_low + x^d t_high (two sparse passes, exact mod 2^64).
//
// The bulk work maps onto two GEMM shapes on CUDA cores (64-bit MACs as
// IMAD.WIDE + 2 IMAD):
//   * many elements times ONE element c:  rows . M_c   (r3_gr_matmul)
//   * sum of many products:  sum_i F_i (x) G_i, i.e. F^T G folded along
//     anti-diagonals                                        (r3_gr_dotsum)
#include "r3_common.cuh"

namespace r3 {

// ---------------------------------------------------------------------------
// polynomial reduction helper (one warp; p has 2D-1 coefficients in smem)
// ---------------------------------------------------------------------------
template <int D>
__device__ void reduce_poly_warp(const u64* p, u64* t, u64 lowterms, u64* out, u64 mask, int lane,
                                 const u64* addend) {
  // t[k] = sum_{j in L} high[k - j],  high[m] = p[D + m], m <= D-2
  constexpr int TLEN = 2 * D + 8;
  for (int k = lane; k < TLEN; k += 32) {
    u64 v = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if ((lowterms >> j) & 1ull) {
        int m = k - j;
        if (m >= 0 && m <= D - 2) v += p[D + m];
      }
    }
    t[k] = v;
  }
  __syncwarp();
  for (int k = lane; k < D; k += 32) {
    u64 v = p[k] - t[k];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if ((lowterms >> j) & 1ull) {
        int m = k - j;  // index into t_high = t[D + m]
        if (m >= 0 && D + m < TLEN) v += t[D + m];
      }
    }
    if (addend) v += addend[k];
    out[k] = v & mask;
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// generic row-wise GR product (warp per row)
// ---------------------------------------------------------------------------
template <int D>
__global__ void gr_mul_kernel(const u64* __restrict__ a, int64_t a_rs, const u64* __restrict__ b, int64_t b_rs,
                              u64* __restrict__ out, int64_t rows, u64 lowterms, u64 mask) {
  constexpr int WARPS = 4;
  __shared__ u64 sa[WARPS][D], sb[WARPS][D], sp[WARPS][2 * D], st[WARPS][2 * D + 8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t row = blockIdx.x * int64_t(WARPS) + w; row < rows; row += int64_t(gridDim.x) * WARPS) {
    for (int k = lane; k < D; k += 32) {
      sa[w][k] = a[row * a_rs + k];
      sb[w][k] = b[row * b_rs + k];
    }
    __syncwarp();
    for (int idx = lane; idx < 2 * D - 1; idx += 32) {
      int lo = idx - (D - 1) > 0 ? idx - (D - 1) : 0;
      int hi = idx < D - 1 ? idx : D - 1;
      u64 acc = 0;
      for (int i = lo; i <= hi; ++i) acc += sa[w][i] * sb[w][idx - i];
      sp[w][idx] = acc;
    }
    __syncwarp();
    reduce_poly_warp<D>(sp[w], st[w], lowterms, out + row * D, mask, lane, nullptr);
  }
}

__global__ void gr_scale_rows_kernel(const u64* __restrict__ s, int64_t s_stride, const u64* __restrict__ g,
                                     int64_t g_rs, u64* __restrict__ out, int64_t rows, int d, u64 mask) {
  const int64_t total = rows * d;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += stride) {
    int64_t r = i / d;
    int k = int(i - r * d);
    out[i] = (s[r * s_stride] * g[r * g_rs + k]) & mask;
  }
}

// M row j = x^j * c mod f  (one block, D threads, D sequential shifts)
__global__ void gr_mulmat_kernel(const u64* __restrict__ c, int d, u64 lowterms, u64* __restrict__ M) {
  __shared__ u64 row[64];
  const int k = threadIdx.x;
  if (k < d) row[k] = c[k];
  __syncthreads();
  for (int j = 0; j < d; ++j) {
    u64 cur = k < d ? row[k] : 0;
    if (k < d) M[j * d + k] = cur;
    u64 top = row[d - 1];
    u64 prev = (k >= 1 && k < d) ? row[k - 1] : 0;
    __syncthreads();
    if (k < d) {
      u64 nv = prev;
      if ((lowterms >> k) & 1ull) nv -= top;
      row[k] = nv;
    }
    __syncthreads();
  }
}

// Public per-level values of one reduction from the opened even point ze
// (verify._Quad, verify.py:215-241): one warp computes
//   u = ze >> 1,  l0 = (ze-1)(u-1),  l1 = ze(2-ze),  l2 = u(ze-1)   (mod f, width)
// and writes out = [l0, l1 - l0, l2, 1 - ze]; with Mo/Mz non-null also the
// multiplication matrices of (1 - ze) and ze (gr_mulmat_kernel's rows).
template <int D>
__device__ void warp_gr_mul(const u64* a, const u64* b, u64* p, u64* t, u64 lowterms, u64* out, u64 mask,
                            int lane) {
  for (int idx = lane; idx < 2 * D - 1; idx += 32) {
    const int lo = idx - (D - 1) > 0 ? idx - (D - 1) : 0;
    const int hi = idx < D - 1 ? idx : D - 1;
    u64 acc = 0;
    for (int i = lo; i <= hi; ++i) acc += a[i] * b[idx - i];
    p[idx] = acc;
  }
  __syncwarp();
  reduce_poly_warp<D>(p, t, lowterms, out, mask, lane, nullptr);
}

template <int D>
__global__ void gr_quad_kernel(const u64* __restrict__ ze, u64 lowterms, u64 mask, u64* __restrict__ out,
                               u64* __restrict__ Mo, u64* __restrict__ Mz) {
  __shared__ u64 z[D], zm1[D], um1[D], tmz[D], u[D], om[D], p[2 * D], t[2 * D + 8], l0[D], l1[D];
  const int lane = threadIdx.x;
  for (int k = lane; k < D; k += 32) {
    const u64 zk = ze[k];
    const u64 e = k == 0 ? 1ull : 0ull;
    z[k] = zk;
    u[k] = zk >> 1;
    zm1[k] = (zk - e) & mask;
    um1[k] = ((zk >> 1) - e) & mask;
    tmz[k] = (2 * e - zk) & mask;
    om[k] = (e - zk) & mask;
  }
  __syncwarp();
  warp_gr_mul<D>(zm1, um1, p, t, lowterms, l0, mask, lane);
  warp_gr_mul<D>(z, tmz, p, t, lowterms, l1, mask, lane);
  warp_gr_mul<D>(u, zm1, p, t, lowterms, out + 2 * D, mask, lane);
  for (int k = lane; k < D; k += 32) {
    out[k] = l0[k];
    out[D + k] = (l1[k] - l0[k]) & mask;
    out[3 * D + k] = om[k];
  }
  if (Mo == nullptr) return;
  // rows j = x^j * c mod f for c = 1 - ze (Mo) and c = ze (Mz)
  __shared__ u64 ro[D], rz[D];
  for (int k = lane; k < D; k += 32) {
    ro[k] = om[k];
    rz[k] = z[k];
  }
  __syncwarp();
  for (int j = 0; j < D; ++j) {
    u64 no[(D + 31) / 32], nz[(D + 31) / 32];
    const u64 to = ro[D - 1], tz = rz[D - 1];
#pragma unroll
    for (int q = 0; q < (D + 31) / 32; ++q) {
      const int k = lane + 32 * q;
      if (k < D) {
        Mo[j * D + k] = ro[k];
        Mz[j * D + k] = rz[k];
        u64 vo = k >= 1 ? ro[k - 1] : 0, vz = k >= 1 ? rz[k - 1] : 0;
        if ((lowterms >> k) & 1ull) {
          vo -= to;
          vz -= tz;
        }
        no[q] = vo;
        nz[q] = vz;
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < (D + 31) / 32; ++q) {
      const int k = lane + 32 * q;
      if (k < D) {
        ro[k] = no[q];
        rz[k] = nz[q];
      }
    }
    __syncwarp();
  }
}

// out[i] = A_i . M (+ C_i): 256 threads, 4x4 register tiles, whole M in smem.
template <int D>
__global__ void __launch_bounds__(256)
gr_matmul_kernel(LinOperand A, const u64* __restrict__ M, int has_c, LinOperand C, u64* __restrict__ out,
                 int64_t rows, u64 mask) {
  constexpr int CG = D / 4;          // column groups of 4
  constexpr int RG = 256 / CG;       // row groups of 4
  constexpr int BM = RG * 4;
  extern __shared__ __align__(16) u64 smem[];
  u64* sM = smem;                    // D*D
  u64* sA = smem + D * D;            // BM*D
  for (int i = threadIdx.x; i < D * D; i += 256) sM[i] = M[i];
  const int tx = threadIdx.x % CG, ty = threadIdx.x / CG;
  for (int64_t r0 = blockIdx.x * int64_t(BM); r0 < rows; r0 += int64_t(gridDim.x) * BM) {
    __syncthreads();
    for (int i = threadIdx.x; i < BM * D; i += 256) {
      int r = i / D, k = i % D;
      int64_t row = r0 + r;
      sA[i] = row < rows ? lin_load(A, row, k) : 0ull;
    }
    __syncthreads();
    u64 acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0;
#pragma unroll 4
    for (int k = 0; k < D; ++k) {
      u64 av[4], mv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sA[(ty * 4 + a) * D + k];
      ulonglong2 m01 = *reinterpret_cast<const ulonglong2*>(&sM[k * D + tx * 4]);
      ulonglong2 m23 = *reinterpret_cast<const ulonglong2*>(&sM[k * D + tx * 4 + 2]);
      mv[0] = m01.x; mv[1] = m01.y; mv[2] = m23.x; mv[3] = m23.y;
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] += av[a] * mv[b];
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      int64_t row = r0 + ty * 4 + a;
      if (row >= rows) continue;
      u64 v[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        v[b] = acc[a][b];
        if (has_c) v[b] += lin_load(C, row, tx * 4 + b);
        v[b] &= mask;
      }
      u64* o = out + row * D + tx * 4;
      reinterpret_cast<ulonglong2*>(o)[0] = make_ulonglong2(v[0], v[1]);
      reinterpret_cast<ulonglong2*>(o)[1] = make_ulonglong2(v[2], v[3]);
    }
  }
}

// acc[0..2D-2] += sum_i F_i (x) G_i.  Each thread owns a 4x4 tile of the
// D x D outer-product sum; 256/(D/4)^2 thread groups split the rows.  Rows
// stream through a double-buffered smem stage: the next BK rows (lazy linear
// combinations of up to 4 views each) are loaded into registers while the
// current stage is multiplied.
template <int D>
__global__ void __launch_bounds__(256, 2)
gr_dotsum_kernel(LinOperand F, LinOperand G, int64_t rows, int64_t rows_per_block, u64* __restrict__ acc) {
  constexpr int CG = D / 4;
  constexpr int TILES = CG * CG;
  constexpr int GROUPS = 256 / TILES;
  constexpr int BK = 32;
  constexpr int PER = BK * D / 256;     // elements of F (and of G) per thread per stage
  extern __shared__ __align__(16) u64 dsm[];
  u64* sF = dsm;                        // [2][BK*D]
  u64* sG = dsm + 2 * BK * D;           // [2][BK*D]
  u64* sP = dsm + 4 * BK * D;           // [2D]
  const int grp = threadIdx.x / TILES;
  const int tile = threadIdx.x % TILES;
  const int ta = tile / CG, tb = tile % CG;
  for (int i = threadIdx.x; i < 2 * D; i += 256) sP[i] = 0;
  u64 s[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) s[a][b] = 0;
  const int64_t r_begin = blockIdx.x * rows_per_block;
  const int64_t r_end = min(rows, r_begin + rows_per_block);
  u64 pf[PER], pg[PER];
  auto fetch = [&](int64_t r0) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int i = threadIdx.x + 256 * q;
      const int64_t row = r0 + i / D;
      const bool ok = row < r_end;
      pf[q] = ok ? lin_load(F, row, i % D) : 0ull;
      pg[q] = ok ? lin_load(G, row, i % D) : 0ull;
    }
  };
  int buf = 0;
  if (r_begin < r_end) fetch(r_begin);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += BK) {
    u64* cF = sF + buf * BK * D;
    u64* cG = sG + buf * BK * D;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      cF[threadIdx.x + 256 * q] = pf[q];
      cG[threadIdx.x + 256 * q] = pg[q];
    }
    __syncthreads();
    if (r0 + BK < r_end) fetch(r0 + BK);
    for (int r = grp; r < BK; r += GROUPS) {
      ulonglong2 f01 = *reinterpret_cast<const ulonglong2*>(&cF[r * D + ta * 4]);
      ulonglong2 f23 = *reinterpret_cast<const ulonglong2*>(&cF[r * D + ta * 4 + 2]);
      ulonglong2 g01 = *reinterpret_cast<const ulonglong2*>(&cG[r * D + tb * 4]);
      ulonglong2 g23 = *reinterpret_cast<const ulonglong2*>(&cG[r * D + tb * 4 + 2]);
      u64 fv[4] = {f01.x, f01.y, f23.x, f23.y};
      u64 gv[4] = {g01.x, g01.y, g23.x, g23.y};
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) s[a][b] += fv[a] * gv[b];
    }
    buf ^= 1;
  }
  __syncthreads();
  // fold the tile along anti-diagonals: coefficient (ta*4+a) + (tb*4+b)
  u64 diag[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) diag[q] = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) diag[a + b] += s[a][b];
  const int base = ta * 4 + tb * 4;
#pragma unroll
  for (int q = 0; q < 7; ++q)
    if (base + q < 2 * D - 1 && diag[q]) atomicAdd(&sP[base + q], diag[q]);
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * D - 1; i += 256)
    if (sP[i]) atomicAdd(acc + i, sP[i]);
}

// ---------------------------------------------------------------------------
// One party's h(1)/h(2) folds of a dense reduction level in ONE pass
// (verify.py:223-230 + gates.py:100-106).  With F from the x side and G from
// the y side, the party's leg products are
//     h = FA (x) (c3 GA + c1 GB) + c2 FB (x) GA
// (P0: FA = x.total, GA = y.total, c3 = 1; P1: c1 = c2 = -1 over m / s1;
//  P2: c3 = 1, c1 = c2 = -1 over m / s2), with F = f1 (odd rows) for h(1)
// and F = 2 f1 - f0 for h(2) (same for G).  The four component arrays stream
// through a 3-stage cp.async pipeline (odd and even row of each pair, zero
// fill past the end = the reference's zero pad); threads [0,256) own 4x4
// tiles of h(1), threads [256,512) of h(2).
// ---------------------------------------------------------------------------
struct LevelArrays {
  const u64* xa;
  const u64* xb;
  const u64* ya;
  const u64* yb;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// pairs per pipeline stage: every (4x4 tile, pair-group) thread busy
__host__ __device__ constexpr int lf_bk(int D) { return D == 16 ? 32 : 8; }

template <int D, int ROLE>
__global__ void __launch_bounds__(512, 1)
level_fold_kernel(LevelArrays A, int64_t N, int64_t pairs_per_block, u64* __restrict__ out1, u64* __restrict__ out2) {
  constexpr int NARR = ROLE == 0 ? 2 : 4;  // xa, ya (+ xb, yb)
  constexpr int BK = lf_bk(D);             // pairs per stage
  constexpr int STAGES = 3;
  constexpr int ROWW = 2 * D;              // odd + even row, in words
  constexpr int STAGE_WORDS = NARR * BK * ROWW;
  constexpr int CG = D / 4, TILES = CG * CG, GROUPS = 256 / TILES;
  extern __shared__ __align__(16) u64 sm[];
  u64* stage_base = sm;                              // [STAGES][NARR][BK][2][D]
  u64* sP = sm + STAGES * STAGE_WORDS;               // [2][2D]
  const int tid = threadIdx.x;
  const int which = tid >> 8;                        // 0: h(1), 1: h(2)
  const int t8 = tid & 255;
  const int grp = t8 / TILES, tile = t8 % TILES;
  const int ta = tile / CG, tb = tile % CG;
  for (int i = tid; i < 4 * D; i += 512) sP[i] = 0;
  const int64_t npairs = (N + 1) / 2;
  const int64_t p_begin = blockIdx.x * pairs_per_block;
  const int64_t p_end = min(npairs, p_begin + pairs_per_block);
  const int64_t nst = (p_end - p_begin + BK - 1) / BK;
  const u64* arr[4] = {A.xa, A.ya, A.xb, A.yb};

  auto issue = [&](int64_t st) {
    if (st < nst) {
      u64* dst = stage_base + (st % STAGES) * STAGE_WORDS;
      constexpr int CHUNKS = STAGE_WORDS / 2;        // 16-byte chunks
      for (int c = tid; c < CHUNKS; c += 512) {
        const int w = c * 2;
        const int a = w / (BK * ROWW);
        const int rem = w % (BK * ROWW);
        const int pr = rem / ROWW, half = (rem % ROWW) / D, k = rem % D;  // half 0: odd, 1: even
        const int64_t pj = p_begin + st * BK + pr;
        const int64_t row = 2 * pj + (half == 0 ? 1 : 0);
        const bool ok = pj < p_end && row < N;
        cp_async16(dst + w, ok ? arr[a] + row * D + k : arr[a], ok);
      }
    }
    cp_async_commit();
  };

  u64 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0;

  for (int s0 = 0; s0 < STAGES - 1; ++s0) issue(s0);
  for (int64_t st = 0; st < nst; ++st) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    issue(st + STAGES - 1);
    const u64* cur = stage_base + (st % STAGES) * STAGE_WORDS;
    for (int pr = grp; pr < BK; pr += GROUPS) {
      // F/G vectors (4 coefficients each) for this thread's tile
      u64 fa[4], fb[4], ga[4], gb[4];
      auto ld4 = [&](int a, int half, int off, u64 (&v)[4]) {
        const u64* src = cur + (a * BK + pr) * ROWW + half * D + off;
        ulonglong2 v01 = *reinterpret_cast<const ulonglong2*>(src);
        ulonglong2 v23 = *reinterpret_cast<const ulonglong2*>(src + 2);
        v[0] = v01.x; v[1] = v01.y; v[2] = v23.x; v[3] = v23.y;
      };
      ld4(0, 0, ta * 4, fa);
      ld4(1, 0, tb * 4, ga);
      if (ROLE != 0) {
        ld4(2, 0, ta * 4, fb);
        ld4(3, 0, tb * 4, gb);
      }
      if (which == 1) {  // f2 = 2 f1 - f0
        u64 e[4];
        ld4(0, 1, ta * 4, e);
#pragma unroll
        for (int q = 0; q < 4; ++q) fa[q] = 2 * fa[q] - e[q];
        ld4(1, 1, tb * 4, e);
#pragma unroll
        for (int q = 0; q < 4; ++q) ga[q] = 2 * ga[q] - e[q];
        if (ROLE != 0) {
          ld4(2, 1, ta * 4, e);
#pragma unroll
          for (int q = 0; q < 4; ++q) fb[q] = 2 * fb[q] - e[q];
          ld4(3, 1, tb * 4, e);
#pragma unroll
          for (int q = 0; q < 4; ++q) gb[q] = 2 * gb[q] - e[q];
        }
      }
      if (ROLE == 0) {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] += fa[a] * ga[b];
      } else {
        u64 gp[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) gp[q] = (ROLE == 2 ? ga[q] : 0ull) - gb[q];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] += fa[a] * gp[b] - fb[a] * ga[b];
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  u64 diag[7];
#pragma unroll
  for (int q = 0; q < 7; ++q) diag[q] = 0;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) diag[a + b] += acc[a][b];
  const int base = ta * 4 + tb * 4;
  u64* myP = sP + which * 2 * D;
#pragma unroll
  for (int q = 0; q < 7; ++q)
    if (base + q < 2 * D - 1 && diag[q]) atomicAdd(&myP[base + q], diag[q]);
  __syncthreads();
  for (int i = tid; i < 2 * D - 1; i += 512) {
    if (sP[i]) atomicAdd(out1 + i, sP[i]);
    if (sP[2 * D + i]) atomicAdd(out2 + i, sP[2 * D + i]);
  }
}

// small-degree fallback (D in {1,2,4}): thread per row, full product in regs
template <int D>
__global__ void gr_dotsum_small_kernel(LinOperand F, LinOperand G, int64_t rows, u64* __restrict__ acc) {
  u64 p[2 * D - 1];
#pragma unroll
  for (int q = 0; q < 2 * D - 1; ++q) p[q] = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t row = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; row < rows; row += stride) {
    u64 f[D], g[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      f[k] = lin_load(F, row, k);
      g[k] = lin_load(G, row, k);
    }
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) p[a + b] += f[a] * g[b];
  }
#pragma unroll
  for (int q = 0; q < 2 * D - 1; ++q) {
    u64 v = p[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(acc + q, v);
  }
}

template <int D>
__global__ void reduce_poly_kernel(const u64* __restrict__ acc, u64 lowterms, u64* __restrict__ out, u64 mask,
                                   int accumulate) {
  __shared__ u64 sp[2 * D], st[2 * D + 8], sadd[D];
  const int lane = threadIdx.x;
  for (int i = lane; i < 2 * D; i += 32) sp[i] = i < 2 * D - 1 ? acc[i] : 0;
  for (int i = lane; i < D; i += 32) sadd[i] = accumulate ? out[i] : 0;
  __syncwarp();
  reduce_poly_warp<D>(sp, st, lowterms, out, mask, lane, sadd);
}

// ---------------------------------------------------------------------------
// fused verification stages over compressed operands
// ---------------------------------------------------------------------------
struct CompPtrs {
  const u64* p[8];
};
struct OutPtrs {
  u64* p[8];
};

// i / n for i >= 0: a shift for power-of-two n (uniform branch)
__device__ __forceinline__ int64_t qdiv64(int64_t i, int64_t n) {
  return (n & (n - 1)) == 0 ? (i >> (__ffsll(n) - 1)) : i / n;
}

__device__ __forceinline__ int64_t comp_off(int64_t i, int64_t n, int64_t ks, int64_t ls) {
  int64_t l = qdiv64(i, n);
  return (i - l * n) * ks + l * ls;
}

// out[c][k] += sum_l comps[c][l*stride] * pw[l][k]
template <int D>
__global__ void __launch_bounds__(256)
powsum_kernel(int ncomp, CompPtrs comps, int64_t stride, int64_t lanes, const u64* __restrict__ pw,
              u64* __restrict__ out) {
  constexpr int RP = 256 / D;  // rows in parallel
  __shared__ u64 red[8][256];
  const int k = threadIdx.x % D, rp = threadIdx.x / D;
  u64 acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = 0;
  for (int64_t l = blockIdx.x * int64_t(RP) + rp; l < lanes; l += int64_t(gridDim.x) * RP) {
    u64 w = __ldg(pw + l * D + k);
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < ncomp) acc[c] += __ldg(comps.p[c] + l * stride) * w;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < ncomp) red[c][threadIdx.x] = acc[c];
  __syncthreads();
  if (rp == 0) {
    for (int c = 0; c < ncomp; ++c) {
      u64 v = 0;
      for (int q = 0; q < RP; ++q) v += red[c][q * D + k];
      atomicAdd(out + c * D + k, v);
    }
  }
}

// h(1)/h(2) folds at level 1 (see r3b200.h).  Terms: coef[t] * fold(x_t, y_t).
template <int D>
__global__ void __launch_bounds__(256)
l1_fold_kernel(int nterms, const int64_t* __restrict__ coef_dev, CompPtrs xc, CompPtrs yc, int64_t N,
               int64_t n, int64_t ks, int64_t ls, const u64* __restrict__ pw, u64* __restrict__ out_h1,
               u64* __restrict__ out_h2, int64_t coef0, int64_t coef1, int64_t coef2, int64_t coef3) {
  constexpr int RP = 256 / D;
  __shared__ u64 red1[256], red2[256];
  const int k = threadIdx.x % D, rp = threadIdx.x / D;
  const int64_t coefs[4] = {coef0, coef1, coef2, coef3};
  const int64_t npairs = (N + 1) / 2;
  u64 h1 = 0, h2 = 0;
  for (int64_t j = blockIdx.x * int64_t(RP) + rp; j < npairs; j += int64_t(gridDim.x) * RP) {
    const int64_t i0 = 2 * j, i1 = 2 * j + 1;
    const bool has1 = i1 < N;
    const int64_t o0 = comp_off(i0, n, ks, ls);
    const int64_t o1 = has1 ? comp_off(i1, n, ks, ls) : 0;
    u64 c1 = 0, c2o = 0, c2e = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (t < nterms) {
        const u64 cf = u64(coefs[t]);
        const u64 x0 = __ldg(xc.p[t] + o0), y0 = __ldg(yc.p[t] + o0);
        const u64 x1 = has1 ? __ldg(xc.p[t] + o1) : 0ull, y1 = has1 ? __ldg(yc.p[t] + o1) : 0ull;
        const u64 g2 = 2 * y1 - y0;
        c1 += cf * (x1 * y1);
        c2o += cf * (2 * x1 * g2);
        c2e -= cf * (x0 * g2);
      }
    }
    const u64 w0 = __ldg(pw + qdiv64(i0, n) * D + k);
    const u64 w1 = has1 ? __ldg(pw + qdiv64(i1, n) * D + k) : 0ull;
    h1 += c1 * w1;
    h2 += c2o * w1 + c2e * w0;
  }
  red1[threadIdx.x] = h1;
  red2[threadIdx.x] = h2;
  __syncthreads();
  if (rp == 0) {
    u64 v1 = 0, v2 = 0;
    for (int q = 0; q < RP; ++q) {
      v1 += red1[q * D + k];
      v2 += red2[q * D + k];
    }
    atomicAdd(out_h1 + k, v1);
    atomicAdd(out_h2 + k, v2);
  }
}

// Small degrees (d <= 16): one thread per pair.  The scalar leg products
// of a pair are computed once (the D-threads-per-pair form above repeats
// them in every coefficient lane) and the thread accumulates all D
// coefficients of h(1)/h(2) from the two power rows (128-bit loads);
// warp shuffles and one shared-memory pass reduce a block to 2 D atomics.
template <int D>
__global__ void __launch_bounds__(256, 2)
l1_fold_pair_kernel(int nterms, CompPtrs xc, CompPtrs yc, int64_t N, int64_t n, int64_t ks, int64_t ls,
                    const u64* __restrict__ pw, u64* __restrict__ out_h1, u64* __restrict__ out_h2,
                    int64_t coef0, int64_t coef1, int64_t coef2, int64_t coef3) {
  __shared__ u64 part[8][2 * D];
  const int64_t coefs[4] = {coef0, coef1, coef2, coef3};
  const int64_t npairs = (N + 1) / 2;
  u64 h1[D], h2[D];
#pragma unroll
  for (int k = 0; k < D; ++k) h1[k] = h2[k] = 0;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < npairs; j += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i0 = 2 * j, i1 = 2 * j + 1;
    const bool has1 = i1 < N;
    const int64_t o0 = comp_off(i0, n, ks, ls);
    const int64_t o1 = has1 ? comp_off(i1, n, ks, ls) : 0;
    u64 c1 = 0, c2o = 0, c2e = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (t < nterms) {
        const u64 cf = u64(coefs[t]);
        const u64 x0 = __ldg(xc.p[t] + o0), y0 = __ldg(yc.p[t] + o0);
        const u64 x1 = has1 ? __ldg(xc.p[t] + o1) : 0ull, y1 = has1 ? __ldg(yc.p[t] + o1) : 0ull;
        const u64 g2 = 2 * y1 - y0;
        c1 += cf * (x1 * y1);
        c2o += cf * (2 * x1 * g2);
        c2e -= cf * (x0 * g2);
      }
    }
    const ulonglong2* r0 = reinterpret_cast<const ulonglong2*>(pw + qdiv64(i0, n) * D);
    const ulonglong2* r1 = reinterpret_cast<const ulonglong2*>(pw + qdiv64(i1, n) * D);
#pragma unroll
    for (int q = 0; q < D / 2; ++q) {
      const ulonglong2 w0 = __ldg(r0 + q);
      const ulonglong2 w1 = has1 ? __ldg(r1 + q) : make_ulonglong2(0ull, 0ull);
      h1[2 * q] += c1 * w1.x;
      h1[2 * q + 1] += c1 * w1.y;
      h2[2 * q] += c2o * w1.x + c2e * w0.x;
      h2[2 * q + 1] += c2o * w1.y + c2e * w0.y;
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < D; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      h1[k] += __shfl_down_sync(0xffffffffu, h1[k], off);
      h2[k] += __shfl_down_sync(0xffffffffu, h2[k], off);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      part[warp][k] = h1[k];
      part[warp][D + k] = h2[k];
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * D) {
    u64 v = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += part[w][threadIdx.x];
    atomicAdd(threadIdx.x < D ? out_h1 + threadIdx.x : out_h2 + (threadIdx.x - D), v);
  }
}

template <int D>
__global__ void l1_line_x_kernel(int ncomp, CompPtrs xc, int64_t N, int64_t n, int64_t ks, int64_t ls,
                                 const u64* __restrict__ A, const u64* __restrict__ B, int64_t tq, OutPtrs out,
                                 u64 mask) {
  const int64_t npairs = (N + 1) / 2;
  const int64_t total = npairs * D;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += stride) {
    const int64_t j = e / D;
    const int k = int(e - j * D);
    const int64_t i0 = 2 * j, i1 = 2 * j + 1;
    const bool has1 = i1 < N;
    const u64 a = __ldg(A + qdiv64(i0, tq) * D + k);
    const u64 b = has1 ? __ldg(B + qdiv64(i1, tq) * D + k) : 0ull;
    const int64_t o0 = comp_off(i0, n, ks, ls);
    const int64_t o1 = has1 ? comp_off(i1, n, ks, ls) : 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < ncomp) {
        u64 x0 = __ldg(xc.p[c] + o0);
        u64 x1 = has1 ? __ldg(xc.p[c] + o1) : 0ull;
        out.p[c][e] = (x0 * a + x1 * b) & mask;
      }
    }
  }
}

template <int D>
__global__ void l1_line_y_kernel(int ncomp, CompPtrs yc, int64_t N, int64_t n, int64_t ks, int64_t ls,
                                 const u64* __restrict__ a, const u64* __restrict__ b, OutPtrs out, u64 mask) {
  const int64_t npairs = (N + 1) / 2;
  const int64_t total = npairs * D;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += stride) {
    const int64_t j = e / D;
    const int k = int(e - j * D);
    const int64_t i0 = 2 * j, i1 = 2 * j + 1;
    const bool has1 = i1 < N;
    const u64 av = a[k], bv = b[k];
    const int64_t o0 = comp_off(i0, n, ks, ls);
    const int64_t o1 = has1 ? comp_off(i1, n, ks, ls) : 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < ncomp) {
        u64 y0 = __ldg(yc.p[c] + o0);
        u64 y1 = has1 ? __ldg(yc.p[c] + o1) : 0ull;
        out.p[c][e] = (y0 * av + y1 * bv) & mask;
      }
    }
  }
}

__global__ void mask_rows_kernel(u64* out, int64_t n, u64 mask) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] &= mask;
}


// ---------------------------------------------------------------------------
// out[f][row] = sum_t a[t][f][row] * c[t]: a public-weighted combination of
// up to 4 share fields in one launch (the Lagrange recombination
// z' = h0 l0 + h1 l1 + h2 l2 of verify.py:233-236 for every field the party
// holds).  Warp per (field, row); the T products are summed unreduced and
// reduced once.
// ---------------------------------------------------------------------------
struct LincombArgs {
  const u64* a[3][4];
  const u64* c[3];
  u64* out[4];
};

template <int D>
__global__ void gr_lincomb_kernel(LincombArgs args, int k, int nterms, int64_t rows, u64 lowterms, u64 mask) {
  constexpr int WARPS = 4;
  __shared__ u64 sc[3][D];
  __shared__ u64 sa[WARPS][D], sp[WARPS][2 * D], st[WARPS][2 * D + 8];
  for (int i = threadIdx.x; i < 3 * D; i += blockDim.x) {
    const int t = i / D;
    sc[t][i - t * D] = t < nterms ? args.c[t][i - t * D] : 0ull;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t items = rows * k;
  for (int64_t it = blockIdx.x * int64_t(WARPS) + w; it < items; it += int64_t(gridDim.x) * WARPS) {
    const int f = int(it / rows);
    const int64_t row = it - int64_t(f) * rows;
    for (int idx = lane; idx < 2 * D; idx += 32) sp[w][idx] = 0;
    for (int t = 0; t < nterms; ++t) {
      __syncwarp();
      for (int q = lane; q < D; q += 32) sa[w][q] = args.a[t][f][row * D + q];
      __syncwarp();
      for (int idx = lane; idx < 2 * D - 1; idx += 32) {
        const int lo = idx - (D - 1) > 0 ? idx - (D - 1) : 0;
        const int hi = idx < D - 1 ? idx : D - 1;
        u64 acc = 0;
        for (int i = lo; i <= hi; ++i) acc += sa[w][i] * sc[t][idx - i];
        sp[w][idx] += acc;
      }
    }
    __syncwarp();
    reduce_poly_warp<D>(sp[w], st[w], lowterms, args.out[f] + row * D, mask, lane, nullptr);
  }
}

}  // namespace r3

using namespace r3;

static bool valid_d(int d) { return d == 1 || d == 2 || d == 4 || d == 8 || d == 16 || d == 32 || d == 64; }

#define R3_DISPATCH_D(d, KERNEL_CALL)           \
  switch (d) {                                  \
    case 1: { constexpr int D = 1; KERNEL_CALL; } break;   \
    case 2: { constexpr int D = 2; KERNEL_CALL; } break;   \
    case 4: { constexpr int D = 4; KERNEL_CALL; } break;   \
    case 8: { constexpr int D = 8; KERNEL_CALL; } break;   \
    case 16: { constexpr int D = 16; KERNEL_CALL; } break; \
    case 32: { constexpr int D = 32; KERNEL_CALL; } break; \
    case 64: { constexpr int D = 64; KERNEL_CALL; } break; \
  }

static LinOperand to_lin(const r3_lin_operand& o) {
  LinOperand l;
  for (int q = 0; q < 4; ++q) {
    l.p[q] = reinterpret_cast<const u64*>(o.p[q]);
    l.rowstride[q] = o.rowstride[q];
    l.nvalid[q] = o.nvalid[q];
    l.coef[q] = o.coef[q];
  }
  l.nterms = o.nterms;
  return l;
}

extern "C" int r3_gr_mul(const uint64_t* a, int64_t a_rs, const uint64_t* b, int64_t b_rs, uint64_t* out,
                         int64_t rows, int d, uint64_t lowterms, uint64_t mask, void* stream) {
  if (!valid_d(d) || rows < 0) {
    set_error("r3_gr_mul: unsupported degree %d", d);
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  unsigned grid = grid_for(rows, 4, 16);
  cudaStream_t s = as_stream(stream);
  R3_DISPATCH_D(d, (gr_mul_kernel<D><<<grid, 128, 0, s>>>((const u64*)a, a_rs, (const u64*)b, b_rs, (u64*)out,
                                                          rows, lowterms, mask)));
  return check_launch("r3_gr_mul");
}

extern "C" int r3_gr_scale_rows(const uint64_t* s, int64_t s_stride, const uint64_t* g, int64_t g_rs,
                                uint64_t* out, int64_t rows, int d, uint64_t mask, void* stream) {
  if (d < 1 || d > 64 || rows < 0) {
    set_error("r3_gr_scale_rows: bad arguments");
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  gr_scale_rows_kernel<<<grid_for(rows * d, 256), 256, 0, as_stream(stream)>>>(
      (const u64*)s, s_stride, (const u64*)g, g_rs, (u64*)out, rows, d, mask);
  return check_launch("r3_gr_scale_rows");
}

extern "C" int r3_gr_mulmat(const uint64_t* c, int d, uint64_t lowterms, uint64_t* M, void* stream) {
  if (!valid_d(d)) {
    set_error("r3_gr_mulmat: unsupported degree %d", d);
    return R3_ERR_ARG;
  }
  gr_mulmat_kernel<<<1, 64, 0, as_stream(stream)>>>((const u64*)c, d, lowterms, (u64*)M);
  return check_launch("r3_gr_mulmat");
}

extern "C" int r3_gr_matmul(r3_lin_operand A, const uint64_t* M, int has_c, r3_lin_operand C, uint64_t* out,
                            int64_t rows, int d, uint64_t mask, void* stream) {
  if (!(d == 8 || d == 16 || d == 32 || d == 64) || rows < 0 || A.nterms < 1 || A.nterms > 4) {
    set_error("r3_gr_matmul: unsupported degree %d / operand", d);
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  cudaStream_t s = as_stream(stream);
  LinOperand la = to_lin(A), lc = to_lin(C);
  switch (d) {
#define R3_MM(DD)                                                                              \
  case DD: {                                                                                   \
    constexpr int CG = DD / 4, RG = 256 / CG, BM = RG * 4;                                     \
    size_t smem = size_t(DD * DD + BM * DD) * 8;                                               \
    ensure_smem(gr_matmul_kernel<DD>, int(smem));                                                   \
    unsigned grid = grid_for((rows + BM - 1) / BM, 1, 3);                                      \
    gr_matmul_kernel<DD><<<grid, 256, smem, s>>>(la, (const u64*)M, has_c, lc, (u64*)out, rows, \
                                                 mask);                                        \
  } break;
    R3_MM(8)
    R3_MM(16)
    R3_MM(32)
    R3_MM(64)
#undef R3_MM
  }
  return check_launch("r3_gr_matmul");
}

extern "C" int r3_gr_dotsum(r3_lin_operand F, r3_lin_operand G, int64_t rows, int d, uint64_t* acc,
                            void* stream) {
  if (!valid_d(d) || rows < 0 || F.nterms < 1 || G.nterms < 1) {
    set_error("r3_gr_dotsum: bad arguments (d=%d)", d);
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  cudaStream_t s = as_stream(stream);
  LinOperand lf = to_lin(F), lg = to_lin(G);
  if (d <= 4) {
    unsigned grid = grid_for(rows, 256, 4);
    if (d == 1) gr_dotsum_small_kernel<1><<<grid, 256, 0, s>>>(lf, lg, rows, (u64*)acc);
    if (d == 2) gr_dotsum_small_kernel<2><<<grid, 256, 0, s>>>(lf, lg, rows, (u64*)acc);
    if (d == 4) gr_dotsum_small_kernel<4><<<grid, 256, 0, s>>>(lf, lg, rows, (u64*)acc);
    return check_launch("r3_gr_dotsum(small)");
  }
  int64_t blocks = int64_t(num_sms()) * 2;
  int64_t per = (rows + blocks - 1) / blocks;
  if (per < 64) per = 64;
  per = (per + 31) / 32 * 32;
  blocks = (rows + per - 1) / per;
  switch (d) {
#define R3_DS(DD)                                                                                 \
  case DD: {                                                                                      \
    const size_t smem = size_t(4 * 32 * DD + 2 * DD) * 8;                                         \
    ensure_smem(gr_dotsum_kernel<DD>, int(smem));                                                   \
    gr_dotsum_kernel<DD><<<unsigned(blocks), 256, smem, s>>>(lf, lg, rows, per, (u64*)acc);      \
  } break;
    R3_DS(8)
    R3_DS(16)
    R3_DS(32)
    R3_DS(64)
#undef R3_DS
  }
  return check_launch("r3_gr_dotsum");
}

extern "C" int r3_gr_quad(const uint64_t* ze, int d, uint64_t lowterms, uint64_t mask, uint64_t* out,
                          uint64_t* Mo, uint64_t* Mz, void* stream) {
  if (d < 1 || d > 64 || (d & (d - 1)) || ((Mo == nullptr) != (Mz == nullptr))) {
    set_error("r3_gr_quad: bad arguments (d %d)", d);
    return R3_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  R3_DISPATCH_D(d, (gr_quad_kernel<D><<<1, 32, 0, s>>>((const u64*)ze, lowterms, mask, (u64*)out, (u64*)Mo,
                                                        (u64*)Mz)));
  return check_launch("r3_gr_quad");
}

extern "C" int r3_gr_reduce_poly(const uint64_t* acc, int d, uint64_t lowterms, uint64_t* out, uint64_t mask,
                                 int accumulate, void* stream) {
  if (!valid_d(d)) {
    set_error("r3_gr_reduce_poly: unsupported degree %d", d);
    return R3_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  R3_DISPATCH_D(d, (reduce_poly_kernel<D><<<1, 32, 0, s>>>((const u64*)acc, lowterms, (u64*)out, mask,
                                                           accumulate)));
  return check_launch("r3_gr_reduce_poly");
}

// nrows accumulators at acc + i (2d - 1), reduced into out + i d: one warp each
template <int D>
__global__ void reduce_poly_rows_kernel(const u64* __restrict__ acc, u64 lowterms, u64* __restrict__ out,
                                        u64 mask) {
  __shared__ u64 sp[2 * D], st[2 * D + 8], sadd[D];
  const int lane = threadIdx.x;
  const u64* a = acc + int64_t(blockIdx.x) * (2 * D - 1);
  for (int i = lane; i < 2 * D; i += 32) sp[i] = i < 2 * D - 1 ? a[i] : 0;
  for (int i = lane; i < D; i += 32) sadd[i] = 0;
  __syncwarp();
  reduce_poly_warp<D>(sp, st, lowterms, out + int64_t(blockIdx.x) * D, mask, lane, sadd);
}

extern "C" int r3_gr_reduce_poly_rows(const uint64_t* acc, int nrows, int d, uint64_t lowterms, uint64_t* out,
                                      uint64_t mask, void* stream) {
  if (!valid_d(d) || nrows < 0 || (nrows && (!acc || !out))) {
    set_error("r3_gr_reduce_poly_rows: bad arguments (d %d, rows %d)", d, nrows);
    return R3_ERR_ARG;
  }
  if (nrows == 0) return R3_OK;
  cudaStream_t s = as_stream(stream);
  R3_DISPATCH_D(d, (reduce_poly_rows_kernel<D><<<nrows, 32, 0, s>>>((const u64*)acc, lowterms, (u64*)out, mask)));
  return check_launch("r3_gr_reduce_poly_rows");
}

static int finish_mask(u64* out, int64_t n, uint64_t mask, cudaStream_t s) {
  if (mask == ~0ull) return R3_OK;
  mask_rows_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n, mask);
  return check_launch("mask");
}

extern "C" int r3_vfy_powsum(int ncomp, const uint64_t* const* comps, int64_t stride, int64_t lanes,
                             const uint64_t* pw, int d, uint64_t* out, uint64_t mask, void* stream) {
  if (ncomp < 1 || ncomp > 8 || !valid_d(d) || lanes < 0) {
    set_error("r3_vfy_powsum: bad arguments");
    return R3_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(out, 0, size_t(ncomp) * d * 8, s);
  if (e != cudaSuccess) {
    set_error("r3_vfy_powsum: memset: %s", cudaGetErrorString(e));
    return R3_ERR_CUDA;
  }
  if (lanes == 0) return R3_OK;
  CompPtrs cp{};
  for (int c = 0; c < ncomp; ++c) cp.p[c] = reinterpret_cast<const u64*>(comps[c]);
  R3_DISPATCH_D(d, ({
                  constexpr int RP = 256 / D;
                  unsigned grid = grid_for((lanes + RP - 1) / RP, 1, 4);
                  powsum_kernel<D><<<grid, 256, 0, s>>>(ncomp, cp, stride, lanes, (const u64*)pw, (u64*)out);
                }));
  int rc = check_launch("r3_vfy_powsum");
  if (rc) return rc;
  return finish_mask((u64*)out, int64_t(ncomp) * d, mask, s);
}

// Level-0 folds of a dot log (n even): every element of lane l carries the
// same power pw[l], so per lane the pair products reduce to two scalars,
//   C1_l = sum_pairs sum_t c_t x1 y1,  C2_l = sum_pairs sum_t c_t (2 x1 - x0)(2 y1 - y0),
// and h1 = sum_l C1_l pw[l], h2 = sum_l C2_l pw[l] (2 D MACs per lane instead
// of 3 D per pair).  Phase 1: one thread per lane (loads coalesced across
// lanes, element (k, l) at k ks + l ls); phase 2: thread (h, k) of the block
// sums its lanes' scalars times pw[l][k].
template <int D>
__global__ void __launch_bounds__(256)
l1_fold_lanes_kernel(int nterms, CompPtrs xc, CompPtrs yc, int64_t L, int64_t n, int64_t ks, int64_t ls,
                     const u64* __restrict__ pw, u64* __restrict__ out_h1, u64* __restrict__ out_h2,
                     int64_t coef0, int64_t coef1, int64_t coef2, int64_t coef3) {
  __shared__ u64 sC[2][256];
  const int64_t coefs[4] = {coef0, coef1, coef2, coef3};
  u64 acc[(2 * D + 255) / 256];
#pragma unroll
  for (int q = 0; q < (2 * D + 255) / 256; ++q) acc[q] = 0;
  for (int64_t l0 = int64_t(blockIdx.x) * 256; l0 < L; l0 += int64_t(gridDim.x) * 256) {
    const int64_t l = l0 + threadIdx.x;
    u64 c1 = 0, c2 = 0;
    if (l < L) {
      for (int64_t k = 0; k < n; k += 2) {
        const int64_t o0 = k * ks + l * ls, o1 = o0 + ks;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (t < nterms) {
            const u64 cf = u64(coefs[t]);
            const u64 x0 = __ldg(xc.p[t] + o0), y0 = __ldg(yc.p[t] + o0);
            const u64 x1 = __ldg(xc.p[t] + o1), y1 = __ldg(yc.p[t] + o1);
            c1 += cf * (x1 * y1);
            c2 += cf * ((2 * x1 - x0) * (2 * y1 - y0));
          }
        }
      }
    }
    sC[0][threadIdx.x] = c1;
    sC[1][threadIdx.x] = c2;
    __syncthreads();
    const int nl = int(L - l0 < 256 ? L - l0 : 256);
#pragma unroll
    for (int q = 0; q < (2 * D + 255) / 256; ++q) {
      const int e = threadIdx.x + 256 * q;
      if (e < 2 * D) {
        const int h = e / D, kk = e % D;
        u64 a = 0;
        for (int r = 0; r < nl; ++r) a += sC[h][r] * __ldg(pw + (l0 + r) * D + kk);
        acc[q] += a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < (2 * D + 255) / 256; ++q) {
    const int e = threadIdx.x + 256 * q;
    if (e < 2 * D) atomicAdd(reinterpret_cast<unsigned long long*>((e < D ? out_h1 : out_h2) + e % D),
                             (unsigned long long)acc[q]);
  }
}

extern "C" int r3_vfy_l1_fold(int nterms, const int64_t* coef, const uint64_t* const* xc,
                              const uint64_t* const* yc, int64_t N, int64_t n, int64_t ks, int64_t ls,
                              const uint64_t* pw, int d, uint64_t* out_h1, uint64_t* out_h2, uint64_t mask,
                              void* stream) {
  if (nterms < 1 || nterms > 4 || !valid_d(d) || N < 0 || n < 1) {
    set_error("r3_vfy_l1_fold: bad arguments");
    return R3_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(out_h1, 0, size_t(d) * 8, s) != cudaSuccess ||
      cudaMemsetAsync(out_h2, 0, size_t(d) * 8, s) != cudaSuccess) {
    set_error("r3_vfy_l1_fold: memset failed");
    return R3_ERR_CUDA;
  }
  if (N == 0) return R3_OK;
  CompPtrs xp{}, yp{};
  int64_t cf[4] = {0, 0, 0, 0};
  for (int t = 0; t < nterms; ++t) {
    xp.p[t] = reinterpret_cast<const u64*>(xc[t]);
    yp.p[t] = reinterpret_cast<const u64*>(yc[t]);
    cf[t] = coef[t];
  }
  const int64_t npairs = (N + 1) / 2;
  if (n >= 4 && n % 2 == 0 && N % n == 0) {
    // dot log: per-lane scalar sums, one power row per lane
    const int64_t L = N / n;
    R3_DISPATCH_D(d, (l1_fold_lanes_kernel<D><<<grid_for(L, 256, 4), 256, 0, s>>>(
                         nterms, xp, yp, L, n, ks, ls, (const u64*)pw, (u64*)out_h1, (u64*)out_h2, cf[0], cf[1],
                         cf[2], cf[3])));
  } else if (d == 16 || d == 8) {
    const unsigned grid = grid_for(npairs, 256, 4);
    if (d == 16)
      l1_fold_pair_kernel<16><<<grid, 256, 0, s>>>(nterms, xp, yp, N, n, ks, ls, (const u64*)pw, (u64*)out_h1,
                                                   (u64*)out_h2, cf[0], cf[1], cf[2], cf[3]);
    else
      l1_fold_pair_kernel<8><<<grid, 256, 0, s>>>(nterms, xp, yp, N, n, ks, ls, (const u64*)pw, (u64*)out_h1,
                                                  (u64*)out_h2, cf[0], cf[1], cf[2], cf[3]);
  } else {
    R3_DISPATCH_D(d, ({
                    constexpr int RP = 256 / D;
                    unsigned grid = grid_for((npairs + RP - 1) / RP, 1, 4);
                    l1_fold_kernel<D><<<grid, 256, 0, s>>>(nterms, nullptr, xp, yp, N, n, ks, ls, (const u64*)pw,
                                                           (u64*)out_h1, (u64*)out_h2, cf[0], cf[1], cf[2], cf[3]);
                  }));
  }
  int rc = check_launch("r3_vfy_l1_fold");
  if (rc) return rc;
  rc = finish_mask((u64*)out_h1, d, mask, s);
  if (rc) return rc;
  return finish_mask((u64*)out_h2, d, mask, s);
}

extern "C" int r3_vfy_l1_line_x(int ncomp, const uint64_t* const* xc, int64_t N, int64_t n, int64_t ks,
                                int64_t ls, const uint64_t* A, const uint64_t* B, int64_t tq, int d,
                                uint64_t* const* out, uint64_t mask, void* stream) {
  if (ncomp < 1 || ncomp > 8 || !valid_d(d) || N < 0 || n < 1 || tq < 1) {
    set_error("r3_vfy_l1_line_x: bad arguments");
    return R3_ERR_ARG;
  }
  if (N == 0) return R3_OK;
  CompPtrs xp{};
  OutPtrs op{};
  for (int c = 0; c < ncomp; ++c) {
    xp.p[c] = reinterpret_cast<const u64*>(xc[c]);
    op.p[c] = reinterpret_cast<u64*>(out[c]);
  }
  const int64_t total = (N + 1) / 2 * d;
  cudaStream_t s = as_stream(stream);
  R3_DISPATCH_D(d, (l1_line_x_kernel<D><<<grid_for(total, 256), 256, 0, s>>>(
                       ncomp, xp, N, n, ks, ls, (const u64*)A, (const u64*)B, tq, op, mask)));
  return check_launch("r3_vfy_l1_line_x");
}

extern "C" int r3_vfy_l1_line_y(int ncomp, const uint64_t* const* yc, int64_t N, int64_t n, int64_t ks,
                                int64_t ls, const uint64_t* a, const uint64_t* b, int d, uint64_t* const* out,
                                uint64_t mask, void* stream) {
  if (ncomp < 1 || ncomp > 8 || !valid_d(d) || N < 0 || n < 1) {
    set_error("r3_vfy_l1_line_y: bad arguments");
    return R3_ERR_ARG;
  }
  if (N == 0) return R3_OK;
  CompPtrs yp{};
  OutPtrs op{};
  for (int c = 0; c < ncomp; ++c) {
    yp.p[c] = reinterpret_cast<const u64*>(yc[c]);
    op.p[c] = reinterpret_cast<u64*>(out[c]);
  }
  const int64_t total = (N + 1) / 2 * d;
  cudaStream_t s = as_stream(stream);
  R3_DISPATCH_D(d, (l1_line_y_kernel<D><<<grid_for(total, 256), 256, 0, s>>>(
                       ncomp, yp, N, n, ks, ls, (const u64*)a, (const u64*)b, op, mask)));
  return check_launch("r3_vfy_l1_line_y");
}

// tensor-core form of the d = 64 level fold (lf_tc.cu), used from this many
// row pairs up; smaller levels stay on the CUDA cores
int level_fold_tc(int role, const uint64_t* xa, const uint64_t* xb, const uint64_t* ya, const uint64_t* yb,
                  int64_t N, uint64_t* acc1, uint64_t* acc2, cudaStream_t s);
constexpr int64_t kLevelFoldTcMinPairs = 4096;

extern "C" int r3_vfy_level_fold(int role, const uint64_t* xa, const uint64_t* xb, const uint64_t* ya,
                                 const uint64_t* yb, int64_t N, int d, uint64_t* acc1, uint64_t* acc2,
                                 void* stream) {
  if (role < 0 || role > 2 || !(d == 16 || d == 32 || d == 64) || N < 0 || !xa || !ya ||
      (role != 0 && (!xb || !yb))) {
    set_error("r3_vfy_level_fold: bad arguments (role=%d d=%d)", role, d);
    return R3_ERR_ARG;
  }
  if (N == 0) return R3_OK;
  cudaStream_t s = as_stream(stream);
  const uintptr_t align = uintptr_t(xa) | uintptr_t(xb) | uintptr_t(ya) | uintptr_t(yb);
  if (d == 64 && (N + 1) / 2 >= kLevelFoldTcMinPairs && (align & 15) == 0)
    return level_fold_tc(role, xa, xb, ya, yb, N, acc1, acc2, s);
  LevelArrays la{(const u64*)xa, (const u64*)xb, (const u64*)ya, (const u64*)yb};
  const int64_t npairs = (N + 1) / 2;
  int64_t blocks = num_sms();
  int64_t per = (npairs + blocks - 1) / blocks;
  if (per < 32) per = 32;
  per = (per + lf_bk(d) - 1) / lf_bk(d) * lf_bk(d);
  blocks = (npairs + per - 1) / per;
#define R3_LF(DD, RR)                                                                                   \
  {                                                                                                     \
    constexpr int NARR = RR == 0 ? 2 : 4;                                                               \
    const size_t smem = size_t(3 * NARR * lf_bk(DD) * 2 * DD + 4 * DD) * 8;                             \
    ensure_smem(level_fold_kernel<DD, RR>, int(smem));                                                  \
    level_fold_kernel<DD, RR><<<unsigned(blocks), 512, smem, s>>>(la, N, per, (u64*)acc1, (u64*)acc2); \
  }
#define R3_LF_D(DD)                 \
  if (role == 0) R3_LF(DD, 0)       \
  else if (role == 1) R3_LF(DD, 1)  \
  else R3_LF(DD, 2)
  if (d == 16) { R3_LF_D(16) } else if (d == 32) { R3_LF_D(32) } else { R3_LF_D(64) }
#undef R3_LF_D
#undef R3_LF
  return check_launch("r3_vfy_level_fold");
}

extern "C" int r3_gr_lincomb(int k, int nterms, const uint64_t* const* a, const uint64_t* const* c,
                             uint64_t* const* out, int64_t rows, int d, uint64_t lowterms, uint64_t mask,
                             void* stream) {
  if (!valid_d(d) || k < 1 || k > 4 || nterms < 1 || nterms > 3 || rows < 0) {
    set_error("r3_gr_lincomb: bad arguments (k=%d nterms=%d d=%d)", k, nterms, d);
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  LincombArgs args{};
  for (int t = 0; t < nterms; ++t) {
    args.c[t] = reinterpret_cast<const u64*>(c[t]);
    for (int f = 0; f < k; ++f) args.a[t][f] = reinterpret_cast<const u64*>(a[t * k + f]);
  }
  for (int f = 0; f < k; ++f) args.out[f] = reinterpret_cast<u64*>(out[f]);
  unsigned grid = grid_for(rows * k, 4, 16);
  cudaStream_t s = as_stream(stream);
  R3_DISPATCH_D(d, (gr_lincomb_kernel<D><<<grid, 128, 0, s>>>(args, k, nterms, rows, lowterms, mask)));
  return check_launch("r3_gr_lincomb");
}
