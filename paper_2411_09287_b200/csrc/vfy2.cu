// Second reduction of the batch verification straight from the base-ring
// log (verify.py:215-241 applied twice after verify.py:168-179).
//
// After compression and one reduction with challenge zeta_1 every level-1
// element is a public combination of two base elements:
//     x1_i = sum_{a<2} X_{2i+a} pw_{2i+a} w1_a,   y1_i = sum_{b<2} Y_{2i+b} w1_b
// with the level-1 line weights w1_0 = 1 - ze_1, w1_1 = ze_1 (ze = the opened
// even point 2 zeta).
// The second reduction pairs (x1_{2j}, x1_{2j+1}), so with blocks of four
// base elements 4j + a (a < 4) its folds are
//     h(1) = sum_{a,b in {2,3}} [ sum_j s^{ab}_j pw_{4j+a} ] (x) w1_{a&1} w1_{b&1}
//     h(2) = sum_{a,b < 4} alpha_a alpha_b [ sum_j s^{ab}_j pw_{4j+a} ] (x) w1_{a&1} w1_{b&1}
// (alpha = -1 on the even half, 2 on the odd half), where s^{ab}_j are the
// party's scalar leg products sum_t c_t x_t[4j+a] y_t[4j+b].  So the level
// costs 16 scalar-times-GR accumulations per block (r3_vfy_l2_fold) and the
// level-1 vectors are never formed; the 16 public GR weights are applied
// to the 16 accumulators afterwards (tiny).  The level-2 vectors for the
// dense tail are x2_j = sum_a X_{4j+a} V_a[j] with public tables
// V_a[j] = pw_{4j+a} w1_{a&1} w2_{a>>1} (r3_vfy_line_b), y2 likewise with
// constants.
#include "r3_common.cuh"

namespace r3 {

struct Comps8 {
  const u64* p[8];
};
struct Outs8 {
  u64* p[8];
};

// i / n for i >= 0: a shift when n is a power of two (dot logs of ell-bit
// inner products, n = 64), the 64-bit division otherwise (uniform branch)
__device__ __forceinline__ int64_t qdiv(int64_t i, int64_t n) {
  return (n & (n - 1)) == 0 ? (i >> (__ffsll(n) - 1)) : i / n;
}

__device__ __forceinline__ int64_t elem_off(int64_t i, int64_t n, int64_t ks, int64_t ls) {
  const int64_t l = qdiv(i, n);
  return (i - l * n) * ks + l * ls;
}

// acc[(a*4+b)][k] = sum_j s^{ab}_j pw[(4j+a)/n][k]; terms t < nterms:
// s^{ab}_j = sum_t coef_t x_t[4j+a] y_t[4j+b] (elements >= N read as 0).
template <int D>
__global__ void __launch_bounds__(256)
l2_fold_kernel(int nterms, Comps8 xc, Comps8 yc, int64_t c0, int64_t c1, int64_t c2, int64_t N, int64_t n,
               int64_t ks, int64_t ls, const u64* __restrict__ pw, u64* __restrict__ acc_out) {
  constexpr int RP = 256 / D;            // blocks of 4 elements in flight per CTA
  __shared__ u64 sS[RP][16];
  __shared__ u64 red[16][256];
  const int k = threadIdx.x % D, rp = threadIdx.x / D;
  const int64_t coefs[3] = {c0, c1, c2};
  const int64_t nblk = (N + 3) / 4;
  u64 acc[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) acc[q] = 0;
  for (int64_t j0 = int64_t(blockIdx.x) * RP; j0 < nblk; j0 += int64_t(gridDim.x) * RP) {
    const int64_t j = j0 + rp;
    const bool live = j < nblk;
    // the block's 16 scalar products, each computed once
    if (live) {
      for (int q = k; q < 16; q += D) {
        const int a = q >> 2, b = q & 3;
        const int64_t ia = 4 * j + a, ib = 4 * j + b;
        u64 sv = 0;
        if (ia < N && ib < N) {
          const int64_t oa = elem_off(ia, n, ks, ls), ob = elem_off(ib, n, ks, ls);
#pragma unroll
          for (int t = 0; t < 3; ++t)
            if (t < nterms) sv += u64(coefs[t]) * (__ldg(xc.p[t] + oa) * __ldg(yc.p[t] + ob));
        }
        sS[rp][q] = sv;
      }
    }
    __syncthreads();
    if (live) {
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int64_t ia = 4 * j + a;
        const u64 w = ia < N ? __ldg(pw + qdiv(ia, n) * D + k) : 0ull;
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a * 4 + b] += sS[rp][a * 4 + b] * w;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) red[q][threadIdx.x] = acc[q];
  __syncthreads();
  if (rp == 0) {
    for (int q = 0; q < 16; ++q) {
      u64 v = 0;
      for (int r = 0; r < RP; ++r) v += red[q][r * D + k];
      atomicAdd(acc_out + q * D + k, v);
    }
  }
}

// out_c[j] = sum_{a<B} X_c[B j + a] * T_a[row_a(j)], T_a = tabs + a*tab_stride
// with row_a(j) = (B j + a) / tq  (tq = B for multiplication logs, whose
// tables hold one row per block; tq = n for dot logs sharing a power).
// ONE: a multiplication log (n == 1, tq == B): element i sits at i * ls and
// the table row of block j is j -- no 64-bit divisions in the hot loop.
// CPT coefficients per thread (128-bit table loads and output stores: 2 for
// d >= 32, 4 for d = 16 so the broadcast share loads serve more output); the
// component loop is unrolled over the 8 slots so the pointer arrays stay in
// registers / parameter space.
template <int D>
__host__ __device__ constexpr int lb_cpt() { return D == 16 ? 4 : 2; }

template <int D, bool ONE, bool TAB, int BM>
__global__ void __launch_bounds__(256, BM == 16 ? 2 : (BM == 8 ? 3 : 4))
line_b_kernel(int B, int ncomp, Comps8 xc, int64_t N, int64_t n, int64_t ks, int64_t ls,
              const u64* __restrict__ tabs, int64_t tab_stride, int64_t tq, Outs8 out, u64 mask) {
  // Lane (row j, coefficients k..k+CPT-1); the 4 lanes of an aligned quad
  // share j (H is a multiple of 4), lane b of a quad loads the scalars of
  // elements B j + b (+ 4h for blocks of BM = 8) for every component, and the
  // quad exchanges them by shuffles: BM / 4 loads per component per lane, all
  // issued before any store.
  // blocks of eight: at most 4 components per launch (registers for 4 waves)
  constexpr int CPT = lb_cpt<D>(), V = CPT / 2, H = D / CPT, NH = BM / 4, MC = BM >= 8 ? 4 : 8;
  const int64_t nblk = (N + B - 1) / B;
  const int64_t total = nblk * H;
  const int lane = threadIdx.x & 31, bl = lane & 3, quad0 = lane & ~3;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int k = CPT * int((blockIdx.x * int64_t(blockDim.x) + threadIdx.x) % H);   // invariant: H | stride
  ulonglong2 w[BM][V];
  if (!TAB) {   // public constants g (B x D): per lane, loaded once
#pragma unroll
    for (int a = 0; a < BM; ++a)
#pragma unroll
      for (int q = 0; q < V; ++q)
        w[a][q] = a < B ? __ldg(reinterpret_cast<const ulonglong2*>(tabs + a * D + k) + q) : make_ulonglong2(0ull, 0ull);
  }
  for (int64_t e0 = blockIdx.x * int64_t(blockDim.x) + (threadIdx.x & ~31); e0 < total; e0 += stride) {
    const int64_t e = e0 + lane;
    const bool live = e < total;
    const int64_t j = e / H;
    u64 xs[MC][NH];
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const int64_t i = B * j + bl + 4 * h;
      const bool ok = live && bl + 4 * h < B && i < N;
      const int64_t off = ok ? (ONE ? i * ls : elem_off(i, n, ks, ls)) : 0;
#pragma unroll
      for (int c = 0; c < MC; ++c) xs[c][h] = (c < ncomp && ok) ? __ldg(xc.p[c] + off) : 0ull;
    }
    if (TAB) {
#pragma unroll
      for (int a = 0; a < BM; ++a) {
        const int64_t ia = B * j + a;
        const bool oka = live && a < B && ia < N;
        const int64_t row = ONE ? j : qdiv(ia, tq);
#pragma unroll
        for (int q = 0; q < V; ++q)
          w[a][q] = oka ? __ldg(reinterpret_cast<const ulonglong2*>(tabs + a * tab_stride + row * D + k) + q)
                        : make_ulonglong2(0ull, 0ull);
      }
    }
#pragma unroll
    for (int c = 0; c < MC; ++c) {
      if (c < ncomp) {
        ulonglong2 v[V];
#pragma unroll
        for (int q = 0; q < V; ++q) v[q] = make_ulonglong2(0ull, 0ull);
#pragma unroll
        for (int a = 0; a < BM; ++a) {
          const u64 xv = __shfl_sync(0xffffffffu, xs[c][a >> 2], quad0 + (a & 3));
#pragma unroll
          for (int q = 0; q < V; ++q) {
            v[q].x += xv * w[a][q].x;
            v[q].y += xv * w[a][q].y;
          }
        }
        if (live) {
#pragma unroll
          for (int q = 0; q < V; ++q)
            __stcs(reinterpret_cast<ulonglong2*>(out.p[c] + j * D + k) + q,
                   make_ulonglong2(v[q].x & mask, v[q].y & mask));
        }
      }
    }
  }
}

// out_c[j] = sum_{b<B} Y_c[B j + b] * g_b  (public constants g, B x D): the
// TAB = false form of line_b_kernel.

// ---------------------------------------------------------------------------
// One pass over the power table for a multiplication log (n = 1): the z
// power sum (r3_vfy_powsum), the 16 level-2 accumulators (r3_vfy_l2_fold)
// and, derived from those, the level-1 folds (r3_vfy_l1_fold):
//   h1(level 1) = acc[1][1] + acc[3][3]
//   h2(level 1) = sum_{pair (e,o) in {(0,1),(2,3)}} 4acc[o][o] - 2acc[o][e] - 2acc[e][o] + acc[e][e]
// (pairs (4j, 4j+1), (4j+2, 4j+3) of level 1 are the a-pairs of block j).
// None of the accumulators depends on the level-1 challenge, so the table is
// streamed once per party instead of three times.
//
// Warp-tiled: a warp owns TB = 32 consecutive blocks of 4 elements.  Phase A:
// lane L forms block L's 16 scalar leg products and its z values into
// warp-private shared memory.  Phase B: the warp walks the 128 power rows of
// the tile, each lane holding KPL coefficients (D >= 32) or one coefficient
// of one of 32/D rows (D < 32), multiply-accumulating broadcast scalars.
// ---------------------------------------------------------------------------
// One party's operands of the base fold.  Several parties share one launch:
// block b works for party b % np on tile slice b / np, so the np blocks that
// stream the same power-table rows are adjacent (co-resident) and the table
// is read from HBM once for all parties (L2 hits for the others).
struct BaseFoldParty {
  Comps8 xc, yc, zc;
  int64_t coef[3];
  int nterms, nz;
  int64_t zs;
  u64* acc_out;
  u64* z_out;
};
struct BaseFoldArgs {
  BaseFoldParty p[3];
  int np;
};

// Q4: pw holds r^(4j) (one row per block of four elements) instead of every
// power; the kernel then accumulates acc'[a][b] = sum_j s^{ab}_j r^(4j) and
// z'[c][a] = sum_j z_c[4j+a] r^(4j) (z_out laid out (nz, 4, D)), and the
// caller multiplies by r^a -- a quarter of the table traffic.
template <int D, bool Q4>
__global__ void __launch_bounds__(256)
base_fold_kernel(const __grid_constant__ BaseFoldArgs args, int64_t N, const u64* __restrict__ pw) {
  const BaseFoldParty& P = args.p[blockIdx.x % args.np];
  const int nterms = P.nterms, nz = P.nz;
  const int64_t zs = P.zs;
  const Comps8& xc = P.xc;
  const Comps8& yc = P.yc;
  const Comps8& zc = P.zc;
  u64* __restrict__ acc_out = P.acc_out;
  u64* __restrict__ z_out = P.z_out;
  const int64_t slice = blockIdx.x / args.np, nslices = gridDim.x / args.np;
  constexpr int KPL = D >= 32 ? D / 32 : 1;
  constexpr int RPS = D >= 32 ? 1 : 32 / D;
  constexpr int TB = 32;
  constexpr int W = 8;
  __shared__ u64 sS[W][16][TB];
  __shared__ u64 sZ[W][8][TB];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = D >= 32 ? 0 : lane / D;
  const int kb = D >= 32 ? lane : lane % D;
  const int64_t coefs[3] = {P.coef[0], P.coef[1], P.coef[2]};
  constexpr int NZS = Q4 ? 8 : 2;   // z accumulator slots
  u64 acc[16][KPL], zacc[NZS][KPL];
#pragma unroll
  for (int q = 0; q < 16; ++q)
#pragma unroll
    for (int c = 0; c < KPL; ++c) acc[q][c] = 0;
#pragma unroll
  for (int q = 0; q < NZS; ++q)
#pragma unroll
    for (int c = 0; c < KPL; ++c) zacc[q][c] = 0;
  const int64_t nblk = (N + 3) / 4;
  const int64_t ntiles = (nblk + TB - 1) / TB;
  for (int64_t tile = slice * W + w; tile < ntiles; tile += nslices * W) {
    {  // phase A: block j = tile*TB + lane
      const int64_t i0 = 4 * (tile * TB + lane);
      u64 s[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) s[q] = 0;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        if (t < nterms) {
          u64 xv[4], yv[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const bool ok = i0 + a < N;
            xv[a] = ok ? __ldg(xc.p[t] + i0 + a) : 0ull;
            yv[a] = ok ? __ldg(yc.p[t] + i0 + a) : 0ull;
          }
          const u64 cf = u64(coefs[t]);
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            const u64 cx = cf * xv[a];
#pragma unroll
            for (int b = 0; b < 4; ++b) s[a * 4 + b] += cx * yv[b];
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) sS[w][q][lane] = s[q];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c < nz) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
            sZ[w][c * 4 + a][lane] = i0 + a < N ? __ldg(zc.p[c] + (i0 + a) * zs) : 0ull;
        }
      }
    }
    __syncwarp();
    if constexpr (Q4) {
      // phase B (Q4): one table row r^(4j) per element block, prefetched
      u64 wcur[KPL], wnxt[KPL];
      auto load_row = [&](int e, u64 (&wv)[KPL]) {
        const int64_t j = tile * TB + e;
#pragma unroll
        for (int c = 0; c < KPL; ++c) wv[c] = j < nblk ? __ldg(pw + j * D + kb + 32 * c) : 0ull;
      };
      load_row(r, wcur);
      for (int e0 = 0; e0 < TB; e0 += RPS) {
        const int e = e0 + r;
        if (e0 + RPS < TB) load_row(e + RPS, wnxt);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const u64 sv = sS[w][q][e];
#pragma unroll
          for (int c = 0; c < KPL; ++c) acc[q][c] += sv * wcur[c];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < 4 * nz) {
            const u64 zv = sZ[w][q][e];
#pragma unroll
            for (int c = 0; c < KPL; ++c) zacc[q][c] += zv * wcur[c];
          }
        }
#pragma unroll
        for (int c = 0; c < KPL; ++c) wcur[c] = wnxt[c];
      }
    } else {
      // phase B: the 4 power rows of element block e (plus the next block's,
      // prefetched into registers) -- keeps several row loads in flight
      u64 wcur[4][KPL], wnxt[4][KPL];
      auto load_rows = [&](int e, u64 (&wv)[4][KPL]) {
        const int64_t ib = 4 * (tile * TB + e);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < KPL; ++c) wv[a][c] = ib + a < N ? __ldg(pw + (ib + a) * D + kb + 32 * c) : 0ull;
      };
      load_rows(r, wcur);
      for (int e0 = 0; e0 < TB; e0 += RPS) {
        const int e = e0 + r;
        if (e0 + RPS < TB) load_rows(e + RPS, wnxt);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const u64 sv = sS[w][a * 4 + b][e];
#pragma unroll
            for (int c = 0; c < KPL; ++c) acc[a * 4 + b][c] += sv * wcur[a][c];
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (q < nz) {
              const u64 zv = sZ[w][q * 4 + a][e];
#pragma unroll
              for (int c = 0; c < KPL; ++c) zacc[q][c] += zv * wcur[a][c];
            }
          }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < KPL; ++c) wcur[a][c] = wnxt[a][c];
      }
    }
    __syncwarp();
  }
  // lanes holding the same coefficient of different rows (D < 32)
#pragma unroll
  for (int off = D; off < 32; off <<= 1) {
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q][0] += __shfl_xor_sync(0xffffffffu, acc[q][0], off);
#pragma unroll
    for (int q = 0; q < NZS; ++q) zacc[q][0] += __shfl_xor_sync(0xffffffffu, zacc[q][0], off);
  }
  // across the CTA's warps, then one atomic per coefficient
  __syncthreads();
  u64* red = &sS[0][0][0];  // W * 16 * TB = 4096 words >= W * D
  const int nslots = 16 + (Q4 ? 4 : 1) * nz;
  for (int q = 0; q < nslots; ++q) {
    if (r == 0) {
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
        u64 v = 0;
#pragma unroll
        for (int qq = 0; qq < 16; ++qq)
          if (qq == q) v = acc[qq][c];
#pragma unroll
        for (int qq = 0; qq < NZS; ++qq)
          if (16 + qq == q) v = zacc[qq][c];
        red[w * D + kb + 32 * c] = v;
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < D; k += blockDim.x) {
      u64 v = 0;
#pragma unroll
      for (int ww = 0; ww < W; ++ww) v += red[ww * D + k];
      if (q < 16)
        atomicAdd(acc_out + q * D + k, v);
      else
        atomicAdd(z_out + (q - 16) * D + k, v);
    }
    __syncthreads();
  }
}

// level-1 folds from the 16 accumulators (see base_fold_kernel); masks z.
__global__ void base_fold_finish_kernel(int d, int nz, const u64* __restrict__ acc, u64* __restrict__ h1,
                                        u64* __restrict__ h2, u64* __restrict__ z, u64 mask) {
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    const u64* A = acc + k;
#define ACC(a, b) A[((a) * 4 + (b)) * d]
    h1[k] = (ACC(1, 1) + ACC(3, 3)) & mask;
    h2[k] = (4 * ACC(1, 1) - 2 * ACC(1, 0) - 2 * ACC(0, 1) + ACC(0, 0) + 4 * ACC(3, 3) - 2 * ACC(3, 2) -
             2 * ACC(2, 3) + ACC(2, 2)) & mask;
#undef ACC
    for (int c = 0; c < nz; ++c) z[c * d + k] &= mask;
  }
}

}  // namespace r3

using namespace r3;

#define R3_DISPATCH_D2(d, CALL)                                 \
  switch (d) {                                                  \
    case 8: { constexpr int D = 8; CALL; } break;               \
    case 16: { constexpr int D = 16; CALL; } break;             \
    case 32: { constexpr int D = 32; CALL; } break;             \
    case 64: { constexpr int D = 64; CALL; } break;             \
    default: set_error("unsupported degree %d", d); return R3_ERR_ARG; \
  }

// The 16 level-2 accumulators of a dot log (n % 4 == 0): blocks of four never
// straddle a lane and every element of lane l carries pw[l], so
//   acc[a*4+b] = sum_l S^{ab}_l pw[l],  S^{ab}_l = sum_{blocks j of lane l} s^{ab}_j
// -- 16 scalar sums per lane, then 16 D MACs per lane (instead of 16 D per
// block).  Phase 1: one thread per lane (coalesced across lanes); phase 2:
// thread (q, k) of the block sums its lanes' S^q times pw[l][k].
template <int D>
__global__ void __launch_bounds__(256)
l2_fold_lanes_kernel(int nterms, Comps8 xc, Comps8 yc, int64_t c0, int64_t c1, int64_t c2, int64_t L, int64_t n,
                     int64_t ks, int64_t ls, const u64* __restrict__ pw, u64* __restrict__ acc_out) {
  constexpr int NQ = (16 * D + 255) / 256;
  __shared__ u64 sS[16][256];
  const int64_t coefs[3] = {c0, c1, c2};
  u64 acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0;
  for (int64_t l0 = int64_t(blockIdx.x) * 256; l0 < L; l0 += int64_t(gridDim.x) * 256) {
    const int64_t l = l0 + threadIdx.x;
    u64 S[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) S[q] = 0;
    if (l < L) {
      for (int64_t k = 0; k < n; k += 4) {
        const int64_t o = k * ks + l * ls;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          if (t < nterms) {
            u64 xv[4], yv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              xv[a] = __ldg(xc.p[t] + o + a * ks);
              yv[a] = __ldg(yc.p[t] + o + a * ks);
            }
            const u64 cf = u64(coefs[t]);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const u64 cx = cf * xv[a];
#pragma unroll
              for (int b = 0; b < 4; ++b) S[a * 4 + b] += cx * yv[b];
            }
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) sS[q][threadIdx.x] = S[q];
    __syncthreads();
    const int nl = int(L - l0 < 256 ? L - l0 : 256);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int e = threadIdx.x + 256 * q;
      if (e < 16 * D) {
        const int qq = e / D, kk = e % D;
        u64 a = 0;
        for (int r = 0; r < nl; ++r) a += sS[qq][r] * __ldg(pw + (l0 + r) * D + kk);
        acc[q] += a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int e = threadIdx.x + 256 * q;
    if (e < 16 * D) atomicAdd(reinterpret_cast<unsigned long long*>(acc_out + e), (unsigned long long)acc[q]);
  }
}

extern "C" int r3_vfy_l2_fold(int nterms, const int64_t* coef, const uint64_t* const* xc,
                              const uint64_t* const* yc, int64_t N, int64_t n, int64_t ks, int64_t ls,
                              const uint64_t* pw, int d, uint64_t* acc, void* stream) {
  if (nterms < 1 || nterms > 3 || N < 0 || n < 1) {
    set_error("r3_vfy_l2_fold: bad arguments");
    return R3_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(acc, 0, size_t(16) * d * 8, s) != cudaSuccess) {
    set_error("r3_vfy_l2_fold: memset failed");
    return R3_ERR_CUDA;
  }
  if (N == 0) return R3_OK;
  Comps8 xp{}, yp{};
  int64_t cf[3] = {0, 0, 0};
  for (int t = 0; t < nterms; ++t) {
    xp.p[t] = reinterpret_cast<const u64*>(xc[t]);
    yp.p[t] = reinterpret_cast<const u64*>(yc[t]);
    cf[t] = coef[t];
  }
  const int64_t nblk = (N + 3) / 4;
  if (n >= 4 && n % 4 == 0 && N % n == 0) {
    // dot log: per-lane scalar sums, one power row per lane
    const int64_t L = N / n;
    R3_DISPATCH_D2(d, (l2_fold_lanes_kernel<D><<<grid_for(L, 256, 4), 256, 0, s>>>(
                          nterms, xp, yp, cf[0], cf[1], cf[2], L, n, ks, ls, (const u64*)pw, (u64*)acc)));
    return check_launch("r3_vfy_l2_fold");
  }
  R3_DISPATCH_D2(d, ({
                   constexpr int RP = 256 / D;
                   unsigned grid = grid_for((nblk + RP - 1) / RP, 1, 4);
                   l2_fold_kernel<D><<<grid, 256, 0, s>>>(nterms, xp, yp, cf[0], cf[1], cf[2], N, n, ks, ls,
                                                          (const u64*)pw, (u64*)acc);
                 }));
  return check_launch("r3_vfy_l2_fold");
}

extern "C" int r3_vfy_line_b(int B, int ncomp, const uint64_t* const* xc, int64_t N, int64_t n, int64_t ks,
                             int64_t ls, const uint64_t* tabs, int64_t tab_stride, int64_t tq, int d,
                             uint64_t* const* out, uint64_t mask, void* stream) {
  if (B < 1 || B > 16 || ncomp < 1 || ncomp > 8 || N < 0 || n < 1 || tq < 1 ||
      (B > 4 && (n != 1 || tq != B || ncomp > 4))) {
    set_error("r3_vfy_line_b: bad arguments");
    return R3_ERR_ARG;
  }
  if (N == 0) return R3_OK;
  Comps8 xp{};
  Outs8 op{};
  for (int c = 0; c < ncomp; ++c) {
    xp.p[c] = reinterpret_cast<const u64*>(xc[c]);
    op.p[c] = reinterpret_cast<u64*>(out[c]);
  }
  const int64_t total = (N + B - 1) / B * (d / (d == 16 ? 4 : 2));
  cudaStream_t s = as_stream(stream);
  if (n == 1 && tq == B && B > 8) {
    R3_DISPATCH_D2(d, (line_b_kernel<D, true, true, 16><<<grid_for(total, 256), 256, 0, s>>>(
                          B, ncomp, xp, N, n, ks, ls, (const u64*)tabs, tab_stride, tq, op, mask)));
  } else if (n == 1 && tq == B && B > 4) {
    R3_DISPATCH_D2(d, (line_b_kernel<D, true, true, 8><<<grid_for(total, 256), 256, 0, s>>>(
                          B, ncomp, xp, N, n, ks, ls, (const u64*)tabs, tab_stride, tq, op, mask)));
  } else if (n == 1 && tq == B) {
    R3_DISPATCH_D2(d, (line_b_kernel<D, true, true, 4><<<grid_for(total, 256), 256, 0, s>>>(
                          B, ncomp, xp, N, n, ks, ls, (const u64*)tabs, tab_stride, tq, op, mask)));
  } else {
    R3_DISPATCH_D2(d, (line_b_kernel<D, false, true, 4><<<grid_for(total, 256), 256, 0, s>>>(
                          B, ncomp, xp, N, n, ks, ls, (const u64*)tabs, tab_stride, tq, op, mask)));
  }
  return check_launch("r3_vfy_line_b");
}

extern "C" int r3_vfy_line_b_const(int B, int ncomp, const uint64_t* const* yc, int64_t N, int64_t n, int64_t ks,
                                   int64_t ls, const uint64_t* g, int d, uint64_t* const* out, uint64_t mask,
                                   void* stream) {
  if (B < 1 || B > 16 || ncomp < 1 || ncomp > 8 || N < 0 || n < 1 || (B > 4 && (n != 1 || ncomp > 4))) {
    set_error("r3_vfy_line_b_const: bad arguments");
    return R3_ERR_ARG;
  }
  if (N == 0) return R3_OK;
  Comps8 yp{};
  Outs8 op{};
  for (int c = 0; c < ncomp; ++c) {
    yp.p[c] = reinterpret_cast<const u64*>(yc[c]);
    op.p[c] = reinterpret_cast<u64*>(out[c]);
  }
  const int64_t total = (N + B - 1) / B * (d / (d == 16 ? 4 : 2));
  cudaStream_t s = as_stream(stream);
  if (n == 1 && B > 8) {
    R3_DISPATCH_D2(d, (line_b_kernel<D, true, false, 16><<<grid_for(total, 256), 256, 0, s>>>(
                          B, ncomp, yp, N, n, ks, ls, (const u64*)g, 0, B, op, mask)));
  } else if (n == 1 && B > 4) {
    R3_DISPATCH_D2(d, (line_b_kernel<D, true, false, 8><<<grid_for(total, 256), 256, 0, s>>>(
                          B, ncomp, yp, N, n, ks, ls, (const u64*)g, 0, B, op, mask)));
  } else if (n == 1) {
    R3_DISPATCH_D2(d, (line_b_kernel<D, true, false, 4><<<grid_for(total, 256), 256, 0, s>>>(
                          B, ncomp, yp, N, n, ks, ls, (const u64*)g, 0, B, op, mask)));
  } else {
    R3_DISPATCH_D2(d, (line_b_kernel<D, false, false, 4><<<grid_for(total, 256), 256, 0, s>>>(
                          B, ncomp, yp, N, n, ks, ls, (const u64*)g, 0, B, op, mask)));
  }
  return check_launch("r3_vfy_line_b_const");
}

int base_fold_q4_tc(int np, const int* nterms, const int64_t* coef, const uint64_t* const* xc,
                    const uint64_t* const* yc, const int* nz, const uint64_t* const* zc, const int64_t* zs,
                    int64_t N, const uint64_t* pw4, uint64_t* const* acc, uint64_t* const* zraw,
                    cudaStream_t s);

static int base_fold_launch(int np, const int* nterms, const int64_t* coef, const uint64_t* const* xc,
                            const uint64_t* const* yc, const int* nz, const uint64_t* const* zc,
                            const int64_t* zs, int64_t N, const uint64_t* pw, int d, uint64_t* const* acc,
                            uint64_t* const* h1, uint64_t* const* h2, uint64_t* const* zsum, uint64_t mask,
                            cudaStream_t s, bool q4 = false) {
  BaseFoldArgs args{};
  args.np = np;
  for (int q = 0; q < np; ++q) {
    if (nterms[q] < 1 || nterms[q] > 3 || nz[q] < 0 || nz[q] > 2 || zs[q] < 1) {
      set_error("r3_vfy_base_fold: bad arguments");
      return R3_ERR_ARG;
    }
    if (cudaMemsetAsync(acc[q], 0, size_t(16) * d * 8, s) != cudaSuccess ||
        (nz[q] > 0 && cudaMemsetAsync(zsum[q], 0, size_t(nz[q]) * (q4 ? 4 : 1) * d * 8, s) != cudaSuccess)) {
      set_error("r3_vfy_base_fold: memset failed");
      return R3_ERR_CUDA;
    }
    BaseFoldParty& P = args.p[q];
    P.nterms = nterms[q];
    P.nz = nz[q];
    P.zs = zs[q];
    for (int t = 0; t < nterms[q]; ++t) {
      P.xc.p[t] = reinterpret_cast<const u64*>(xc[3 * q + t]);
      P.yc.p[t] = reinterpret_cast<const u64*>(yc[3 * q + t]);
      P.coef[t] = coef[3 * q + t];
    }
    for (int c = 0; c < nz[q]; ++c) P.zc.p[c] = reinterpret_cast<const u64*>(zc[2 * q + c]);
    P.acc_out = reinterpret_cast<u64*>(acc[q]);
    P.z_out = reinterpret_cast<u64*>(zsum[q]);
  }
  if (N > 0 && q4 && d == 64) {
    // tensor-core form (bf_tc.cu) for large logs
    int rc = base_fold_q4_tc(np, nterms, coef, xc, yc, nz, zc, zs, N, pw, acc, zsum, s);
    if (rc >= 0) return rc;
  }
  if (N > 0) {
    const int64_t ntiles = ((N + 3) / 4 + 31) / 32;
    R3_DISPATCH_D2(d, ({
                     unsigned slices = grid_for((ntiles + 7) / 8, 1, 2);
                     if (q4)
                       base_fold_kernel<D, true><<<slices * np, 256, 0, s>>>(args, N, (const u64*)pw);
                     else
                       base_fold_kernel<D, false><<<slices * np, 256, 0, s>>>(args, N, (const u64*)pw);
                   }));
    int rc = check_launch("r3_vfy_base_fold");
    if (rc) return rc;
  }
  if (q4) return R3_OK;   // raw r^(4j) accumulators: the caller applies r^a and finishes
  for (int q = 0; q < np; ++q) {
    base_fold_finish_kernel<<<1, 64, 0, s>>>(d, nz[q], (const u64*)acc[q], (u64*)h1[q], (u64*)h2[q],
                                             (u64*)zsum[q], mask);
    int rc = check_launch("r3_vfy_base_fold(finish)");
    if (rc) return rc;
  }
  return R3_OK;
}

extern "C" int r3_vfy_base_fold(int nterms, const int64_t* coef, const uint64_t* const* xc,
                                const uint64_t* const* yc, int nz, const uint64_t* const* zc, int64_t zs,
                                int64_t N, const uint64_t* pw, int d, uint64_t* acc, uint64_t* h1, uint64_t* h2,
                                uint64_t* zsum, uint64_t mask, void* stream) {
  if (N < 0 || nterms < 1 || nterms > 3 || nz < 0 || nz > 2) {
    set_error("r3_vfy_base_fold: bad arguments");
    return R3_ERR_ARG;
  }
  int64_t cf[3] = {0, 0, 0};
  const uint64_t* xs[3] = {nullptr, nullptr, nullptr};
  const uint64_t* ys[3] = {nullptr, nullptr, nullptr};
  const uint64_t* zz[2] = {nullptr, nullptr};
  for (int t = 0; t < nterms; ++t) {
    cf[t] = coef[t];
    xs[t] = xc[t];
    ys[t] = yc[t];
  }
  for (int c = 0; c < nz; ++c) zz[c] = zc[c];
  return base_fold_launch(1, &nterms, cf, xs, ys, &nz, zz, &zs, N, pw, d, &acc, &h1, &h2, &zsum, mask,
                          as_stream(stream));
}

extern "C" int r3_vfy_base_fold_q4(int np, const int* nterms, const int64_t* coef, const uint64_t* const* xc,
                                   const uint64_t* const* yc, const int* nz, const uint64_t* const* zc,
                                   const int64_t* zs, int64_t N, const uint64_t* pw4, int d,
                                   uint64_t* const* acc, uint64_t* const* zraw, void* stream) {
  if (np < 1 || np > 3 || N < 0) {
    set_error("r3_vfy_base_fold_q4: bad arguments");
    return R3_ERR_ARG;
  }
  return base_fold_launch(np, nterms, coef, xc, yc, nz, zc, zs, N, pw4, d, acc, nullptr, nullptr, zraw, 0,
                          as_stream(stream), true);
}

extern "C" int r3_vfy_base_fold_finish(int d, int nz, const uint64_t* acc, uint64_t* h1, uint64_t* h2,
                                       uint64_t* zsum, uint64_t mask, void* stream) {
  base_fold_finish_kernel<<<1, 64, 0, as_stream(stream)>>>(d, nz, (const u64*)acc, (u64*)h1, (u64*)h2,
                                                           (u64*)zsum, mask);
  return check_launch("r3_vfy_base_fold_finish");
}

extern "C" int r3_vfy_base_fold_multi(int np, const int* nterms, const int64_t* coef, const uint64_t* const* xc,
                                      const uint64_t* const* yc, const int* nz, const uint64_t* const* zc,
                                      const int64_t* zs, int64_t N, const uint64_t* pw, int d,
                                      uint64_t* const* acc, uint64_t* const* h1, uint64_t* const* h2,
                                      uint64_t* const* zsum, uint64_t mask, void* stream) {
  if (np < 1 || np > 3 || N < 0) {
    set_error("r3_vfy_base_fold_multi: bad arguments");
    return R3_ERR_ARG;
  }
  return base_fold_launch(np, nterms, coef, xc, yc, nz, zc, zs, N, pw, d, acc, h1, h2, zsum, mask,
                          as_stream(stream));
}

// ---------------------------------------------------------------------------
// Dot logs with n % 16 == 0, d = 16 (the edaBits inner products of length
// ell: verify.py:182-241 on the consolidated lane-major vector).  Blocks of
// sixteen consecutive elements lie inside one lane and share its power
// r^(P+l), so the folds of the first FOUR reductions come from 256 per-lane
// scalar sums
//   acc[a*16+b] = sum_l S^{ab}_l pw[l],  S^{ab}_l = sum_{blocks j of lane l} sum_t c_t x_t[16j+a] y_t[16j+b]
// (public level weights, verify._block_fold_weights), and the level-4 rows
// are written straight from the base shares (r3_vfy_lane16_line):
//   x: pw[l] (x) sum_a kappa_a x[16j+a],   y: sum_a kappa_a y[16j+a]
// -- the dense tail starts at N/16 rows instead of N/4.
// ---------------------------------------------------------------------------
constexpr int L16_TILE = 16;     // lanes per tile
constexpr int L16_PAD = L16_TILE + 1;

// Leg terms grouped by their x component: sum_t c_t x_t y_t =
// sum_g x_g (sum_k c_gk y_gk) (P2's three terms are two products).
struct L16Groups {
  const u64* x[3];
  const u64* y[3][3];
  int64_t c[3][3];
  int ny[3];
  int ng;
};

template <int D>
__global__ void __launch_bounds__(256, 2)
lane16_fold_kernel(const __grid_constant__ L16Groups G, int64_t L, int64_t n, const u64* __restrict__ pw,
                   u64* __restrict__ acc_out) {
  // thread (a, b): S^{ab} of the tile's lanes in registers, then its D
  // accumulator words; one block of 16 elements per group staged at a time
  // (x, and the group's combined y)
  __shared__ u64 sX[3][16][L16_PAD], sY[3][16][L16_PAD];
  __shared__ u64 sP[L16_TILE][D];
  const int tid = threadIdx.x, a = tid >> 4, b = tid & 15;
  const int ng = G.ng;
  u64 acc[D];
#pragma unroll
  for (int c = 0; c < D; ++c) acc[c] = 0;
  const int64_t ntiles = (L + L16_TILE - 1) / L16_TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t l0 = tile * L16_TILE;
    u64 S[L16_TILE];
#pragma unroll
    for (int q = 0; q < L16_TILE; ++q) S[q] = 0;
    for (int64_t j = 0; j < n; j += 16) {
      for (int e = tid; e < ng * 16 * L16_TILE; e += 256) {
        const int ln = e % L16_TILE, r = (e / L16_TILE) % 16, g = e / (16 * L16_TILE);
        const int64_t l = l0 + ln;
        u64 xv = 0, yv = 0;
        if (l < L) {
          const int64_t off = (j + r) * L + l;
          xv = __ldg(G.x[g] + off);
          yv = u64(G.c[g][0]) * __ldg(G.y[g][0] + off);
          if (G.ny[g] > 1) yv += u64(G.c[g][1]) * __ldg(G.y[g][1] + off);
          if (G.ny[g] > 2) yv += u64(G.c[g][2]) * __ldg(G.y[g][2] + off);
        }
        sX[g][r][ln] = xv;
        sY[g][r][ln] = yv;
      }
      __syncthreads();
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        if (g < ng) {
#pragma unroll
          for (int q = 0; q < L16_TILE; ++q) S[q] += sX[g][a][q] * sY[g][b][q];
        }
      }
      __syncthreads();
    }
    for (int e = tid; e < L16_TILE * D; e += 256) {
      const int64_t l = l0 + e / D;
      sP[e / D][e % D] = l < L ? __ldg(pw + l * D + e % D) : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < L16_TILE; ++q) {
#pragma unroll
      for (int c = 0; c < D; c += 2) {
        const ulonglong2 pv = *reinterpret_cast<const ulonglong2*>(&sP[q][c]);
        acc[c] += S[q] * pv.x;
        acc[c + 1] += S[q] * pv.y;
      }
    }
    __syncthreads();
  }
  u64* dst = acc_out + (a * 16 + b) * D;
#pragma unroll
  for (int c = 0; c < D; ++c) atomicAdd(reinterpret_cast<unsigned long long*>(dst + c), (unsigned long long)acc[c]);
}

// Level-4 rows of one component: row l (n/16) + j of the consolidated
// order holds base elements 16j..16j+15 of lane l.  One thread per row
// (lanes fastest: coalesced base loads); POW multiplies by pw[l] in
// GR(2^64, D) (schoolbook product reduced by t^D = -sum_{k in lowterms} t^k).
template <int D, bool POW>
__global__ void __launch_bounds__(256)
lane16_line_kernel(int ncomp, const __grid_constant__ Comps8 xc, int64_t L, int64_t n, const u64* __restrict__ pw,
                   const u64* __restrict__ kappa, u64 lowterms, const __grid_constant__ Outs8 out, u64 mask) {
  __shared__ __align__(16) u64 sK[16][D];
  for (int e = threadIdx.x; e < 16 * D; e += blockDim.x) sK[e / D][e % D] = kappa[e];
  __syncthreads();
  const int64_t nb = n / 16, rows = L * nb;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t l = i % L, j = i / L;
    u64 p[D];
    if (POW) {
#pragma unroll
      for (int c = 0; c < D; ++c) p[c] = __ldg(pw + l * D + c);
    }
    for (int cp = 0; cp < ncomp; ++cp) {
      u64 u[D];
#pragma unroll
      for (int c = 0; c < D; ++c) u[c] = 0;
#pragma unroll
      for (int a = 0; a < 16; ++a) {
        const u64 v = __ldg(xc.p[cp] + (16 * j + a) * L + l);
#pragma unroll
        for (int c = 0; c < D; c += 2) {     // 128-bit broadcast reads of the constants
          const ulonglong2 kk = *reinterpret_cast<const ulonglong2*>(&sK[a][c]);
          u[c] += v * kk.x;
          u[c + 1] += v * kk.y;
        }
      }
      u64* o = out.p[cp] + (l * nb + j) * D;
      if (POW) {
        u64 pr[2 * D - 1];
#pragma unroll
        for (int k = 0; k < 2 * D - 1; ++k) pr[k] = 0;
#pragma unroll
        for (int x = 0; x < D; ++x) {
#pragma unroll
          for (int y = 0; y < D; ++y) pr[x + y] += p[x] * u[y];
        }
#pragma unroll
        for (int k = 2 * D - 2; k >= D; --k) {
          const u64 top = pr[k];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if ((lowterms >> q) & 1ull) pr[k - D + q] -= top;
        }
#pragma unroll
        for (int c = 0; c < D; c += 2)
          *reinterpret_cast<ulonglong2*>(o + c) = make_ulonglong2(pr[c] & mask, pr[c + 1] & mask);
      } else {
#pragma unroll
        for (int c = 0; c < D; c += 2)
          *reinterpret_cast<ulonglong2*>(o + c) = make_ulonglong2(u[c] & mask, u[c + 1] & mask);
      }
    }
  }
}

extern "C" int r3_vfy_lane16_fold(int nterms, const int64_t* coef, const uint64_t* const* xc,
                                  const uint64_t* const* yc, int64_t L, int64_t n, const uint64_t* pw, int d,
                                  uint64_t* acc, void* stream) {
  if (nterms < 1 || nterms > 3 || L < 0 || n < 16 || n % 16 || d != 16 || !pw || !acc) {
    set_error("r3_vfy_lane16_fold: bad arguments (1 <= nterms <= 3, n %% 16 == 0, d = 16)");
    return R3_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  if (cudaMemsetAsync(acc, 0, size_t(256) * d * 8, s) != cudaSuccess) {
    set_error("r3_vfy_lane16_fold: memset failed");
    return R3_ERR_CUDA;
  }
  if (L == 0) return R3_OK;
  L16Groups G{};
  for (int t = 0; t < nterms; ++t) {
    int g = 0;
    while (g < G.ng && G.x[g] != reinterpret_cast<const u64*>(xc[t])) ++g;
    if (g == G.ng) {
      G.x[g] = reinterpret_cast<const u64*>(xc[t]);
      ++G.ng;
    }
    G.y[g][G.ny[g]] = reinterpret_cast<const u64*>(yc[t]);
    G.c[g][G.ny[g]] = coef[t];
    ++G.ny[g];
  }
  const int64_t tiles = (L + L16_TILE - 1) / L16_TILE;
  const unsigned grid = unsigned(tiles < int64_t(num_sms()) * 2 ? tiles : int64_t(num_sms()) * 2);
  lane16_fold_kernel<16><<<grid, 256, 0, s>>>(G, L, n, (const u64*)pw, (u64*)acc);
  return check_launch("r3_vfy_lane16_fold");
}

extern "C" int r3_vfy_lane16_line(int pow_side, int ncomp, const uint64_t* const* xc, int64_t L, int64_t n,
                                  const uint64_t* pw, const uint64_t* kappa, uint64_t lowterms, int d,
                                  uint64_t* const* out, uint64_t mask, void* stream) {
  if (ncomp < 1 || ncomp > 8 || L < 0 || n < 16 || n % 16 || d != 16 || !kappa || (pow_side && !pw)) {
    set_error("r3_vfy_lane16_line: bad arguments (1 <= ncomp <= 8, n %% 16 == 0, d = 16)");
    return R3_ERR_ARG;
  }
  if (L == 0) return R3_OK;
  Comps8 xp{};
  Outs8 op{};
  for (int c = 0; c < ncomp; ++c) {
    xp.p[c] = reinterpret_cast<const u64*>(xc[c]);
    op.p[c] = reinterpret_cast<u64*>(out[c]);
  }
  cudaStream_t s = as_stream(stream);
  const unsigned grid = grid_for(L * (n / 16), 256, 4);
  if (pow_side)
    lane16_line_kernel<16, true><<<grid, 256, 0, s>>>(ncomp, xp, L, n, (const u64*)pw, (const u64*)kappa, lowterms,
                                                      op, mask);
  else
    lane16_line_kernel<16, false><<<grid, 256, 0, s>>>(ncomp, xp, L, n, nullptr, (const u64*)kappa, lowterms, op,
                                                       mask);
  return check_launch("r3_vfy_lane16_line");
}

// ---------------------------------------------------------------------------
// Level-4 rows of a d = 16 multiplication log with blocks of sixteen
// straight from the base shares, without the sixteen tables r^(16j)
// (r^a kappa_a) (N x 128 B written and read back):
//   x: pw16[j] (x) sum_a c_a x[16j + a]  (c_a = r^a kappa_a),   y: sum_a kappa_a y[16j + a]
// One thread per row: sixteen scalar x GR(2^64, 16) MACs, then (x side) the
// schoolbook product with pw16[j] reduced by t^16 = -sum_{k in lowterms} t^k.
// ---------------------------------------------------------------------------
template <bool POW>
__global__ void __launch_bounds__(256)
mul16_line_kernel(int ncomp, const __grid_constant__ Comps8 xc, int64_t N, const u64* __restrict__ pw,
                  const u64* __restrict__ coef, u64 lowterms, const __grid_constant__ Outs8 out, u64 mask) {
  constexpr int D = 16;
  __shared__ __align__(16) u64 sK[16][D];
  for (int e = threadIdx.x; e < 16 * D; e += blockDim.x) sK[e / D][e % D] = coef[e];
  __syncthreads();
  const int64_t rows = (N + 15) / 16;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < rows; j += int64_t(gridDim.x) * blockDim.x) {
    u64 p[D];
    if (POW) {
#pragma unroll
      for (int c = 0; c < D; c += 2) {
        const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(pw + j * D + c));
        p[c] = v.x, p[c + 1] = v.y;
      }
    }
    const bool full = 16 * j + 16 <= N;
    for (int cp = 0; cp < ncomp; ++cp) {
      const u64* src = xc.p[cp] + 16 * j;
      u64 xv[16];
      if (full && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
        for (int a = 0; a < 16; a += 2) {
          const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(src + a));
          xv[a] = v.x, xv[a + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int a = 0; a < 16; ++a) xv[a] = 16 * j + a < N ? __ldg(src + a) : 0ull;
      }
      u64 u[D];
#pragma unroll
      for (int c = 0; c < D; ++c) u[c] = 0;
#pragma unroll
      for (int a = 0; a < 16; ++a) {
#pragma unroll
        for (int c = 0; c < D; c += 2) {     // 128-bit broadcast reads of the constants
          const ulonglong2 kk = *reinterpret_cast<const ulonglong2*>(&sK[a][c]);
          u[c] += xv[a] * kk.x;
          u[c + 1] += xv[a] * kk.y;
        }
      }
      u64* o = out.p[cp] + j * D;
      if (POW) {
        u64 pr[2 * D - 1];
#pragma unroll
        for (int k = 0; k < 2 * D - 1; ++k) pr[k] = 0;
#pragma unroll
        for (int x = 0; x < D; ++x) {
#pragma unroll
          for (int y = 0; y < D; ++y) pr[x + y] += p[x] * u[y];
        }
#pragma unroll
        for (int k = 2 * D - 2; k >= D; --k) {
          const u64 top = pr[k];
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if ((lowterms >> q) & 1ull) pr[k - D + q] -= top;
        }
#pragma unroll
        for (int c = 0; c < D; c += 2)
          *reinterpret_cast<ulonglong2*>(o + c) = make_ulonglong2(pr[c] & mask, pr[c + 1] & mask);
      } else {
#pragma unroll
        for (int c = 0; c < D; c += 2)
          *reinterpret_cast<ulonglong2*>(o + c) = make_ulonglong2(u[c] & mask, u[c + 1] & mask);
      }
    }
  }
}

extern "C" int r3_vfy_mul16_line(int pow_side, int ncomp, const uint64_t* const* xc, int64_t N, const uint64_t* pw16,
                                 const uint64_t* coef, uint64_t lowterms, int d, uint64_t* const* out, uint64_t mask,
                                 void* stream) {
  if (ncomp < 1 || ncomp > 8 || N < 0 || d != 16 || !coef || (pow_side && !pw16)) {
    set_error("r3_vfy_mul16_line: bad arguments (1 <= ncomp <= 8, d = 16)");
    return R3_ERR_ARG;
  }
  if (N == 0) return R3_OK;
  Comps8 xp{};
  Outs8 op{};
  for (int c = 0; c < ncomp; ++c) {
    xp.p[c] = reinterpret_cast<const u64*>(xc[c]);
    op.p[c] = reinterpret_cast<u64*>(out[c]);
  }
  cudaStream_t s = as_stream(stream);
  const unsigned grid = grid_for((N + 15) / 16, 256, 4);
  if (pow_side)
    mul16_line_kernel<true><<<grid, 256, 0, s>>>(ncomp, xp, N, (const u64*)pw16, (const u64*)coef, lowterms, op,
                                                 mask);
  else
    mul16_line_kernel<false><<<grid, 256, 0, s>>>(ncomp, xp, N, nullptr, (const u64*)coef, lowterms, op, mask);
  return check_launch("r3_vfy_mul16_line");
}
