// Dense-level verification folds on the tensor cores (d = 64).
//
// One reduction level (verify.py:215-241) needs, per party, the leg folds
//   h(1) = sum_i  o_x(i) (x) o_y(i)          h(2) = sum_i  t_x(i) (x) t_y(i)
// over row pairs i = (2i, 2i+1) = (e, o), with t = 2o - e (the line value at
// the point 2, verify.py:229) and (x) the unreduced polynomial product,
// summed over the party's leg terms (gates.py:100-106).  Each is a matrix
// product X^T Y over K = pairs with X, Y the (pairs x 64) views of the o or
// t rows, so only the two products the protocol needs are formed (no
// e (x) o cross blocks).
//
// Byte limbs: a u64 product is the 36 limb products x_p y_q with p + q <= 7
// (kind::i8, u8 x u8 -> s32), weighted 2^(8(p+q)).  The MMA's M = 128 rows
// hold TWO limb planes of x (p = 2j in rows 0-63, p = 2j+1 in rows 64-127;
// the planes are stored contiguously, so the pair is one MN-major operand)
// against the N-concatenated planes y_0..y_(7-2j): column block q lands at
// TMEM column block 2j + q, i.e. block c holds diagonal c in the upper rows
// and diagonal c + 1 in the lower rows, for every j.  Four plane pairs =
// 4 MMAs per product and 32-pair k-block (N = 8, 6, 4, 2 column blocks).
// Every accumulator sums at most 2 limb products per pair where its
// diagonal needs more than 32 bits (c <= 3), so a 16384-pair item is exact.
//
// Work item = (K chunk, leg term, y half): one CTA forms BOTH products of
// its term for 32 of the 64 y features (2 x 8 blocks x 32 = all 512 TMEM
// columns), reading all of x and half of y; the two y-half siblings are
// adjacent in the grid and do identical work, so they stream x in lock
// step and the second read of each x tile is an L2 hit (DRAM bytes = the
// distinct operand bytes).  Warps 0-3: epilogue (TMEM lane quadrants);
// warps 4-15: converters (swizzled TMA boxes -> o and t rows, B = c0 Y0 +
// c1 Y1 formed on the fly -> limb planes in shared memory); warp 16: TMA
// producer; warp 17: MMA issuer.
#include "tc_common.cuh"

namespace r3 {

constexpr int LF_BK = 32;                        // pairs per k-block (one i8 MMA K step)
constexpr int LF_A_PLANE = 64 * LF_BK;           // one x limb plane (64 features): 2 KB
constexpr int LF_B_PLANE = 32 * LF_BK;           // one y-half limb plane (32 features): 1 KB
constexpr int LF_A_TILE = 8 * LF_A_PLANE;        // 16 KB per product
constexpr int LF_B_TILE = 8 * LF_B_PLANE;        // 8 KB per product
constexpr int LF_LIMB = 2 * (LF_A_TILE + LF_B_TILE);  // o and t operands: 48 KB
constexpr int LF_BOX = 16 * 8 * LF_BK;           // one TMA box: 16 u64 x 32 pair rows = 4 KB
constexpr int LF_RAW = 16 * LF_BOX;              // x 8 boxes + y0 4 + y1 4 = 64 KB
constexpr int LF_STAGES = 2;
constexpr int LF_CONV = 12 * 32;                 // 256 A tasks + 128 B tasks per k-block
constexpr int LF_THREADS = 4 * 32 + LF_CONV + 2 * 32;
constexpr int LF_OFF_LIMB = LF_STAGES * LF_RAW;
constexpr int LF_OFF_BAR = LF_OFF_LIMB + LF_STAGES * LF_LIMB;
constexpr int LF_SMEM = LF_OFF_BAR + 256 + 1024;  // + alignment slack
constexpr int64_t LF_MAX_K = 16384;              // exact-accumulation bound (pairs per item)

// Pair-view tensor maps of one operand vector (row p = rows 2p, 2p+1, 128
// u64): lo covers ceil(rows/2) pairs (the even row, features 0..63), hi
// floor(rows/2) pairs (the odd row, features 64..127).  Rows past a map's
// extent are zero-filled by the TMA unit.
struct LfVec {
  CUtensorMap lo, hi;
};

// One leg term: x (x) (c0 y0 + c1 y1) (y1 < 0: none), added to party
// `out`'s two folds.
struct LfTerm {
  int x, y0, y1;
  u64 c0, c1;
  int out;
};

// Up to the three simulated parties' terms in one launch (honest joint
// sessions: P0 1, P1 2, P2 2 terms over 7 distinct vectors, m shared by P1
// and P2); the items of a chunk are adjacent, so a vector read by several
// terms comes from HBM about once.
struct LfArgs {
  LfVec v[8];
  LfTerm t[5];
  u64* acc1[3];
  u64* acc2[3];
  int nterms;
  int64_t rows, npairs, kc, nchunks;
};

__device__ __forceinline__ void lf_named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// v += coef * (o, or 2 o - e for the t operand) over one 16-u64 box row,
// one 16-byte swizzled chunk at a time (few live registers); MODE 0: coef
// = 1, 1: coef = -1, 2: general
template <int MODE>
__device__ __forceinline__ void lf_accum_row(const uint8_t* ro, const uint8_t* re, bool t, int sw, u64 coef,
                                             u64 (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    ulonglong2 x = *reinterpret_cast<const ulonglong2*>(ro + ((q ^ sw) << 4));
    if (t) {
      const ulonglong2 e = *reinterpret_cast<const ulonglong2*>(re + ((q ^ sw) << 4));
      x.x = 2 * x.x - e.x;
      x.y = 2 * x.y - e.y;
    }
    if (MODE == 0) {
      v[2 * q] += x.x;
      v[2 * q + 1] += x.y;
    } else if (MODE == 1) {
      v[2 * q] -= x.x;
      v[2 * q + 1] -= x.y;
    } else {
      v[2 * q] += coef * x.x;
      v[2 * q + 1] += coef * x.y;
    }
  }
}

__device__ __forceinline__ void lf_accum(const uint8_t* ro, const uint8_t* re, bool t, int sw, u64 coef,
                                         u64 (&v)[16]) {
  if (coef == 1ull)
    lf_accum_row<0>(ro, re, t, sw, coef, v);
  else if (coef == ~0ull)
    lf_accum_row<1>(ro, re, t, sw, coef, v);
  else
    lf_accum_row<2>(ro, re, t, sw, coef, v);
}

__global__ void __launch_bounds__(LF_THREADS, 1)
level_fold_tc_kernel(const __grid_constant__ LfArgs args) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself (keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sRaw = smem;
  uint8_t* sLimb = smem + LF_OFF_LIMB;             // stage: A_o, A_t, B_o, B_t
  u64* red = reinterpret_cast<u64*>(smem);         // epilogue only (raw stages are idle by then)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LF_OFF_BAR);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = bars + LF_STAGES;
  uint64_t* full = bars + 2 * LF_STAGES;
  uint64_t* empty = bars + 3 * LF_STAGES;
  uint64_t* tfull = bars + 4 * LF_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // work item: the y-half siblings are adjacent, then the terms of a chunk
  const int64_t item = blockIdx.x;
  const int yh = int(item & 1);
  const int term = int((item >> 1) % args.nterms);
  const int64_t chunk = (item >> 1) / args.nterms;
  const LfTerm& T = args.t[term];
  const int64_t p0 = chunk * args.kc;
  const int64_t p1 = min(args.npairs, p0 + args.kc);
  const int64_t nkb = (p1 - p0 + LF_BK - 1) / LF_BK;
  const int nyv = T.y1 >= 0 ? 2 : 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < LF_STAGES; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], LF_CONV);
      mbar_init(&full[s], LF_CONV);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4 + 12) {
    // ---------------- TMA producer.  Raw stage: boxes 0-3 x odd row, 4-7 x
    // even row, 8-9 y0 odd (this half), 10-11 y0 even, 12-15 likewise y1
    if (lane == 0) {
      const LfVec& X = args.v[T.x];
      const LfVec& Y0 = args.v[T.y0];
      const LfVec& Y1 = args.v[T.y1 >= 0 ? T.y1 : T.y0];
      for (int64_t kb = 0; kb < nkb; ++kb) {
        const int st = int(kb % LF_STAGES);
        if (kb >= LF_STAGES) mbar_wait(&raw_empty[st], uint32_t((kb / LF_STAGES - 1) & 1));
        const int y = int(p0 + kb * LF_BK);
        uint8_t* dst = sRaw + st * LF_RAW;
        mbar_expect_tx(&raw_full[st], uint32_t((8 + 4 * nyv) * LF_BOX));
        for (int c = 0; c < 4; ++c) {
          tma_load_2d(dst + c * LF_BOX, &X.hi, 64 + c * 16, y, &raw_full[st]);
          tma_load_2d(dst + (4 + c) * LF_BOX, &X.lo, c * 16, y, &raw_full[st]);
        }
        for (int c = 0; c < 2; ++c) {
          tma_load_2d(dst + (8 + c) * LF_BOX, &Y0.hi, 64 + yh * 32 + c * 16, y, &raw_full[st]);
          tma_load_2d(dst + (10 + c) * LF_BOX, &Y0.lo, yh * 32 + c * 16, y, &raw_full[st]);
          if (nyv > 1) {
            tma_load_2d(dst + (12 + c) * LF_BOX, &Y1.hi, 64 + yh * 32 + c * 16, y, &raw_full[st]);
            tma_load_2d(dst + (14 + c) * LF_BOX, &Y1.lo, yh * 32 + c * 16, y, &raw_full[st]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 16) {
    // ---------------- converters: thread = (operand, product o|t, pair row k, 16-feature chunk c)
    const int lt = threadIdx.x - 128;
    const bool isA = lt < 256;
    const int k = lt & 31;
    const int c = isA ? ((lt >> 5) & 3) : ((lt >> 5) & 1);
    const int tt = isA ? (lt >> 7) : ((lt - 256) >> 6);
    const int sw = k & 7;
    for (int64_t kb = 0; kb < nkb; ++kb) {
      const int st = int(kb % LF_STAGES);
      mbar_wait(&raw_full[st], uint32_t((kb / LF_STAGES) & 1));
      const bool ok = p0 + kb * LF_BK + k < p1;   // pairs of the next chunk read as zero
      const uint8_t* raw = sRaw + st * LF_RAW + k * 128;
      u64 v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = 0;
      if (isA) {
        lf_accum_row<0>(raw + c * LF_BOX, raw + (4 + c) * LF_BOX, tt, sw, 1ull, v);
      } else {
        lf_accum(raw + (8 + c) * LF_BOX, raw + (10 + c) * LF_BOX, tt, sw, T.c0, v);
        if (nyv > 1) lf_accum(raw + (12 + c) * LF_BOX, raw + (14 + c) * LF_BOX, tt, sw, T.c1, v);
      }
      fence_async_smem();   // generic-proxy reads before the next TMA write (WAR)
      mbar_arrive(&raw_empty[st]);
      if (!ok) {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = 0;
      }
      uint4 pk[8];
      split_limbs16(v, pk);
      if (kb >= LF_STAGES) mbar_wait(&empty[st], uint32_t((kb / LF_STAGES - 1) & 1));
      // MN-major no-swizzle core layout: chunk stride 512 B, k-row stride 16 B
      uint8_t* base = sLimb + st * LF_LIMB;
      uint8_t* dst = isA ? base + tt * LF_A_TILE : base + 2 * LF_A_TILE + tt * LF_B_TILE;
      const int plane = isA ? LF_A_PLANE : LF_B_PLANE;
      const uint32_t off = uint32_t(c * 512 + k * 16);
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(dst + i * plane + off) = pk[i];
      fence_async_smem();
      mbar_arrive(&full[st]);
    }
  } else if (warp == 4 + 12 + 1) {
    // ---------------- MMA issuer
    constexpr uint32_t IDESC_M128 = idesc_u8(128, 0) | (1u << 15) | (1u << 16);  // A, B MN-major; N set per MMA
    for (int64_t kb = 0; kb < nkb; ++kb) {
      const int st = int(kb % LF_STAGES);
      mbar_wait(&full[st], uint32_t((kb / LF_STAGES) & 1));
      tc_fence_after();
      if (lane == 0) {
        const uint32_t base = smem_u32(sLimb + st * LF_LIMB);
        // product o|t: x planes (2j, 2j+1) against y planes 0..7-2j,
        // N-concatenated: column block q -> TMEM block 2j + q of the
        // product's 256 columns (diagonal 2j + q upper rows, +1 lower rows)
#pragma unroll
        for (int tt = 0; tt < 2; ++tt) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t ad = umma_desc(base + uint32_t(tt * LF_A_TILE + 2 * j * LF_A_PLANE), 128, 512);
            const uint64_t bd = umma_desc(base + uint32_t(2 * LF_A_TILE + tt * LF_B_TILE), 128, 512);
            const int nn = 32 * (8 - 2 * j);
            mma_u8(tmem + uint32_t(tt * 256 + 64 * j), ad, bd, IDESC_M128 | (uint32_t(nn >> 3) << 17),
                   (kb == 0 && j == 0) ? 0u : 1u);
          }
        }
        mma_commit(&empty[st]);
      }
      __syncwarp();
    }
    if (lane == 0) mma_commit(tfull);
    __syncwarp();
  } else if (warp < 4) {
    // ---------------- epilogue: TMEM lane m = (plane parity h, feature a) of x
    if (nkb > 0) {
      mbar_wait(tfull, 0);
      tc_fence_after();
      // every TMA load has been consumed: the raw stages are free for red
      red[threadIdx.x] = 0;
      red[128 + threadIdx.x] = 0;
      lf_named_sync(1, 128);
      const int m = warp * 32 + lane;
      const int h = m >> 6, a = m & 63;
      const uint32_t lane_base = tmem + (uint32_t(warp * 32) << 16);
#pragma unroll 1
      for (int cb = 0; cb < 64; cb += 8) {
        const int tt = cb >> 5, b0 = cb & 31;
        uint32_t v[8][8];
#pragma unroll
        for (int s = 0; s < 8; ++s) tmem_ld8(lane_base + uint32_t(tt * 256 + s * 32 + b0), v[s]);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const u64 P = h == 0 ? recombine8(v[0][q], v[1][q], v[2][q], v[3][q], v[4][q], v[5][q], v[6][q], v[7][q])
                               : recombine8(0u, v[0][q], v[1][q], v[2][q], v[3][q], v[4][q], v[5][q], v[6][q]);
          atomicAdd(reinterpret_cast<unsigned long long*>(red + tt * 128 + a + yh * 32 + b0 + q),
                    (unsigned long long)P);
        }
      }
      tc_fence_before();
      lf_named_sync(1, 128);
      const int t = threadIdx.x;
      if (t < 127) {
        atomicAdd(reinterpret_cast<unsigned long long*>(args.acc1[T.out] + t), (unsigned long long)red[t]);
        atomicAdd(reinterpret_cast<unsigned long long*>(args.acc2[T.out] + t), (unsigned long long)red[128 + t]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace r3

using namespace r3;

static bool lf_vec(LfVec& V, const uint64_t* a, int64_t rows) {
  const int64_t ceilp = (rows + 1) / 2, floorp = rows / 2;
  // a pair-view map with no rows (rows == 1, odd half) is given one row of
  // width 64, so every odd-row box is out of range and reads as zero
  bool ok = make_rows_tmap(&V.lo, a, ceilp, 128, LF_BK, 128);
  ok = ok && (floorp > 0 ? make_rows_tmap(&V.hi, a, floorp, 128, LF_BK, 128)
                         : make_rows_tmap(&V.hi, a, 1, 128, LF_BK, 64));
  return ok;
}

int lf_launch(LfArgs& args, int64_t N, cudaStream_t s);

// Called by r3_vfy_level_fold for d == 64 (same contract).
int level_fold_tc(int role, const uint64_t* xa, const uint64_t* xb, const uint64_t* ya, const uint64_t* yb,
                  int64_t N, uint64_t* acc1, uint64_t* acc2, cudaStream_t s) {
  if (N <= 1) return -1;   // caller's CUDA-core path (a lone row has no odd half)
  LfArgs args{};
  const u64 M1 = ~0ull;  // -1
  // vectors 0..3 = xa, xb, ya, yb
  bool ok = lf_vec(args.v[0], xa, N) && lf_vec(args.v[2], ya, N);
  if (role != 0) ok = ok && lf_vec(args.v[1], xb, N) && lf_vec(args.v[3], yb, N);
  if (!ok) {
    set_error("r3_vfy_level_fold(tc): cuTensorMapEncodeTiled failed");
    return R3_ERR_CUDA;
  }
  if (role == 0) {  // P0: s_x (x) s_y
    args.t[0] = LfTerm{0, 2, -1, 1, 0, 0};
    args.nterms = 1;
  } else if (role == 1) {  // -(m_x s_y) - (s_x m_y)
    args.t[0] = LfTerm{0, 3, -1, M1, 0, 0};
    args.t[1] = LfTerm{1, 2, -1, M1, 0, 0};
    args.nterms = 2;
  } else {  // m_x (m_y - s_y) - s_x m_y
    args.t[0] = LfTerm{0, 2, 3, 1, M1, 0};
    args.t[1] = LfTerm{1, 2, -1, M1, 0, 0};
    args.nterms = 2;
  }
  args.acc1[0] = reinterpret_cast<u64*>(acc1);
  args.acc2[0] = reinterpret_cast<u64*>(acc2);
  return lf_launch(args, N, s);
}

// All three parties in one launch: P0 total (x, y), P1 (m, s1), P2 (s2; m
// shared with P1) -- vectors 0 tx, 1 ty, 2 mx, 3 my, 4 s1x, 5 s1y, 6 s2x, 7
// s2y; acc1 / acc2 of party r at acc1[r] / acc2[r].
extern "C" int r3_vfy_level_fold_joint(const uint64_t* tx, const uint64_t* ty, const uint64_t* mx,
                                       const uint64_t* my, const uint64_t* s1x, const uint64_t* s1y,
                                       const uint64_t* s2x, const uint64_t* s2y, int64_t N, uint64_t* const* acc1,
                                       uint64_t* const* acc2, void* stream) {
  if (N <= 1 || !tx || !ty || !mx || !my || !s1x || !s1y || !s2x || !s2y || !acc1 || !acc2) {
    set_error("r3_vfy_level_fold_joint: bad arguments (N %lld)", (long long)N);
    return R3_ERR_ARG;
  }
  LfArgs args{};
  const u64 M1 = ~0ull;
  const uint64_t* vs[8] = {tx, ty, mx, my, s1x, s1y, s2x, s2y};
  for (int i = 0; i < 8; ++i) {
    if (!lf_vec(args.v[i], vs[i], N)) {
      set_error("r3_vfy_level_fold_joint: cuTensorMapEncodeTiled failed");
      return R3_ERR_CUDA;
    }
  }
  cudaStream_t s = as_stream(stream);
  for (int r = 0; r < 3; ++r) {
    args.acc1[r] = reinterpret_cast<u64*>(acc1[r]);
    args.acc2[r] = reinterpret_cast<u64*>(acc2[r]);
    if (cudaMemsetAsync(acc1[r], 0, 127 * 8, s) != cudaSuccess || cudaMemsetAsync(acc2[r], 0, 127 * 8, s) != cudaSuccess) {
      set_error("r3_vfy_level_fold_joint: memset failed");
      return R3_ERR_CUDA;
    }
  }
  // P1's terms next to P2's (m_x / m_y shared), P0's first
  args.t[0] = LfTerm{0, 1, -1, 1, 0, 0};        // P0: s_x (x) s_y
  args.t[1] = LfTerm{2, 5, -1, M1, 0, 1};       // P1: -(m_x s1_y)
  args.t[2] = LfTerm{2, 3, 7, 1, M1, 2};        // P2: m_x (m_y - s2_y)
  args.t[3] = LfTerm{4, 3, -1, M1, 0, 1};       // P1: -(s1_x m_y)
  args.t[4] = LfTerm{6, 3, -1, M1, 0, 2};       // P2: -(s2_x m_y)
  args.nterms = 5;
  return lf_launch(args, N, s);
}

int lf_launch(LfArgs& args, int64_t N, cudaStream_t s) {
  args.rows = N;
  args.npairs = (N + 1) / 2;
  int64_t nchunks = (args.npairs + LF_MAX_K - 1) / LF_MAX_K;
  const int64_t per_chunk_items = 2 * args.nterms;
  const int64_t waves = (nchunks * per_chunk_items + num_sms() - 1) / num_sms();
  int64_t want = waves * num_sms() / per_chunk_items;  // fill the last wave
  const int64_t min_kc = 8 * LF_BK;
  if (want * min_kc > args.npairs) want = (args.npairs + min_kc - 1) / min_kc;
  if (want > nchunks) nchunks = want;
  int64_t kc = (args.npairs + nchunks - 1) / nchunks;
  kc = (kc + LF_BK - 1) / LF_BK * LF_BK;
  nchunks = (args.npairs + kc - 1) / kc;
  args.kc = kc;
  args.nchunks = nchunks;
  ensure_smem(level_fold_tc_kernel, LF_SMEM);
  const unsigned grid = unsigned(nchunks * per_chunk_items);
  level_fold_tc_kernel<<<grid, LF_THREADS, LF_SMEM, s>>>(args);
  return check_launch("r3_vfy_level_fold(tc)");
}
