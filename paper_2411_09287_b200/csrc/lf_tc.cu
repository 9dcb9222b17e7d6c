// Dense-level verification folds on the tensor cores (d = 64).
//
// One reduction level (verify.py:215-241) needs, per party, the leg folds
//   h(1) = sum_i  x_o(i) (x) y_o(i)          h(2) = sum_i  t_x(i) (x) t_y(i)
// over row pairs i = (2i, 2i+1) = (e, o), with t = 2o - e and (x) the
// unreduced polynomial product, summed over the party's leg terms
// (gates.py:100-106).  Writing P_uv[a][b] = sum_i u_x(i)[a] v_y(i)[b] for
// u, v in {e, o}:
//   h(1)[c] = sum_{a+b=c} P_oo[a][b]
//   h(2)[c] = sum_{a+b=c} (4 P_oo - 2 P_oe - 2 P_eo + P_ee)[a][b]
// and [P_ee P_eo; P_oe P_oo] is ONE matrix product X^T Y with X, Y the
// component arrays viewed as (pairs x 128): M = 128 (both halves of x),
// N = 64 (one half of y per CTA), K = pairs.  Both operands are MN-major in
// that view (features contiguous), so the loaders only split u64 words into
// byte-limb planes -- no transposition.  Each u64 product runs as the 36
// limb products (kind::i8, p + q <= 7) accumulated per diagonal p + q in 8
// TMEM accumulators (8 x 64 of the 512 columns), issued as 12 MMAs of
// N = 64 (8 - p) against N-concatenated B planes; a CTA's K range is <= 16384
// pairs so every diagonal is exact mod 2^32 where it matters (tc.cu).  The
// epilogue recombines the diagonals in u64, applies the (u, v) weights and
// folds the anti-diagonals into the 2d-1 output words.
//
// Work item = (leg term, K chunk, y half).  Warps 0-3: epilogue (TMEM lane
// quadrants); warps 4-15: converters (swizzled TMA boxes -> limb planes in
// shared memory, B operand = c0 Y0 + c1 Y1 formed on the fly); warp 16: TMA
// producer; warp 17: MMA issuer.
#include "tc_common.cuh"

namespace r3 {

constexpr int LF_BM = 128, LF_BN = 64, LF_BK = 32;
constexpr int LF_A_PLANE = LF_BM * LF_BK;        // 4 KB
constexpr int LF_B_PLANE = LF_BN * LF_BK;        // 2 KB
constexpr int LF_A_TILE = 8 * LF_A_PLANE;        // 32 KB of limb planes
constexpr int LF_B_TILE = 8 * LF_B_PLANE;        // 16 KB
constexpr int LF_BOX = 16 * 8 * LF_BK;           // one TMA box: 16 u64 x 32 pair rows = 4 KB
constexpr int LF_RAW = 16 * LF_BOX;              // A 8 boxes + B0 4 + B1 4 = 64 KB
constexpr int LF_STAGES = 2;
constexpr int LF_CONV = 12 * 32;                 // 256 A tasks + 128 B tasks per k-block
constexpr int LF_THREADS = 4 * 32 + LF_CONV + 2 * 32;
constexpr int LF_OFF_LIMB = LF_STAGES * LF_RAW;
constexpr int LF_OFF_BAR = LF_OFF_LIMB + LF_STAGES * (LF_A_TILE + LF_B_TILE);
constexpr int LF_SMEM = LF_OFF_BAR + 256 + 1024;  // + alignment slack
constexpr int64_t LF_MAX_K = 16384;              // exact-accumulation bound (pairs per item)

// Tensor maps of one leg term over the pair view (row p = rows 2p, 2p+1 of
// the component, 128 u64): A_lo covers ceil(rows/2) pairs (features 0..63),
// A_hi floor(rows/2) pairs (features 64..127, the odd row); B maps likewise
// per y half.  Rows past a map's extent are zero-filled by the TMA unit.
struct LfTerm {
  CUtensorMap a_lo, a_hi, b0[2], b1[2];
  u64 c0, c1;
  int has_b1;
};

struct LfArgs {
  LfTerm t[2];
  int nterms;
  int64_t rows, npairs, kc, nchunks;
};

__device__ __forceinline__ void lf_named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// 16 u64 of one swizzled TMA box row -> 8 planes of 16 bytes (byte i of each)
__device__ __forceinline__ void lf_read_row(const uint8_t* row, int sw, u64 (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(row + ((q ^ sw) << 4));
    v[2 * q] = x.x;
    v[2 * q + 1] = x.y;
  }
}

__device__ __forceinline__ void lf_split16(const u64 (&v)[16], uint4 (&out)[8]) {
  uint32_t w[32];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    w[2 * q] = uint32_t(v[q]);
    w[2 * q + 1] = uint32_t(v[q] >> 32);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int hiw = i >> 2, bi = i & 3;
    out[i].x = gather_byte(w[0 + hiw], w[2 + hiw], w[4 + hiw], w[6 + hiw], bi);
    out[i].y = gather_byte(w[8 + hiw], w[10 + hiw], w[12 + hiw], w[14 + hiw], bi);
    out[i].z = gather_byte(w[16 + hiw], w[18 + hiw], w[20 + hiw], w[22 + hiw], bi);
    out[i].w = gather_byte(w[24 + hiw], w[26 + hiw], w[28 + hiw], w[30 + hiw], bi);
  }
}

__global__ void __launch_bounds__(LF_THREADS, 1)
level_fold_tc_kernel(const __grid_constant__ LfArgs args, u64* __restrict__ acc1, u64* __restrict__ acc2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sRaw = smem;
  uint8_t* sA = smem + LF_OFF_LIMB;
  uint8_t* sB = sA + LF_STAGES * LF_A_TILE;
  u64* red1 = reinterpret_cast<u64*>(smem);        // epilogue only (raw stages are idle by then)
  u64* red2 = red1 + 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LF_OFF_BAR);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = bars + LF_STAGES;
  uint64_t* full = bars + 2 * LF_STAGES;
  uint64_t* empty = bars + 3 * LF_STAGES;
  uint64_t* tfull = bars + 4 * LF_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // work item
  const int64_t item = blockIdx.x;
  const int half = int(item & 1);
  const int64_t chunk = (item >> 1) % args.nchunks;
  const int term = int((item >> 1) / args.nchunks);
  const LfTerm& T = args.t[term];
  const int64_t p0 = chunk * args.kc;
  const int64_t p1 = min(args.npairs, p0 + args.kc);
  const int64_t nkb = (p1 - p0 + LF_BK - 1) / LF_BK;
  const int nbox = 8 + 4 + (T.has_b1 ? 4 : 0);

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
    // ---------------- TMA producer
    if (lane == 0) {
      for (int64_t kb = 0; kb < nkb; ++kb) {
        const int st = int(kb % LF_STAGES);
        if (kb >= LF_STAGES) mbar_wait(&raw_empty[st], uint32_t((kb / LF_STAGES - 1) & 1));
        const int y = int(p0 + kb * LF_BK);
        uint8_t* dst = sRaw + st * LF_RAW;
        mbar_expect_tx(&raw_full[st], uint32_t(nbox * LF_BOX));
        for (int c = 0; c < 8; ++c) tma_load_2d(dst + c * LF_BOX, c < 4 ? &T.a_lo : &T.a_hi, c * 16, y, &raw_full[st]);
        for (int c = 0; c < 4; ++c)
          tma_load_2d(dst + (8 + c) * LF_BOX, &T.b0[half], half * 64 + c * 16, y, &raw_full[st]);
        if (T.has_b1)
          for (int c = 0; c < 4; ++c)
            tma_load_2d(dst + (12 + c) * LF_BOX, &T.b1[half], half * 64 + c * 16, y, &raw_full[st]);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 16) {
    // ---------------- converters: thread = (pair row k of the k-block, 16-feature chunk c)
    const int lt = threadIdx.x - 128;
    const bool isA = lt < 256;
    const int k = lt & 31;
    const int c = isA ? (lt >> 5) : ((lt - 256) >> 5);
    const int sw = k & 7;
    for (int64_t kb = 0; kb < nkb; ++kb) {
      const int st = int(kb % LF_STAGES);
      mbar_wait(&raw_full[st], uint32_t((kb / LF_STAGES) & 1));
      const bool ok = p0 + kb * LF_BK + k < p1;   // pairs of the next chunk read as zero
      const uint8_t* raw = sRaw + st * LF_RAW;
      u64 v[16];
      if (isA) {
        lf_read_row(raw + c * LF_BOX + k * 128, sw, v);
      } else {
        lf_read_row(raw + (8 + c) * LF_BOX + k * 128, sw, v);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] *= T.c0;
        if (T.has_b1) {
          u64 w[16];
          lf_read_row(raw + (12 + c) * LF_BOX + k * 128, sw, w);
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] += T.c1 * w[q];
        }
      }
      fence_async_smem();   // generic-proxy reads before the next TMA write (WAR)
      mbar_arrive(&raw_empty[st]);
      if (!ok) {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = 0;
      }
      uint4 pk[8];
      lf_split16(v, pk);
      if (kb >= LF_STAGES) mbar_wait(&empty[st], uint32_t((kb / LF_STAGES - 1) & 1));
      // MN-major no-swizzle core layout: chunk stride 512 B, k-row stride 16 B
      uint8_t* dst = isA ? sA + st * LF_A_TILE : sB + st * LF_B_TILE;
      const int plane = isA ? LF_A_PLANE : LF_B_PLANE;
      const uint32_t off = uint32_t(c * 512 + k * 16);
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(dst + i * plane + off) = pk[i];
      fence_async_smem();
      mbar_arrive(&full[st]);
    }
  } else if (warp == 4 + 12 + 1) {
    // ---------------- MMA issuer
    constexpr uint32_t IDESC_M128 = idesc_u8(LF_BM, 0) | (1u << 15) | (1u << 16);  // A, B MN-major; N set per MMA
    for (int64_t kb = 0; kb < nkb; ++kb) {
      const int st = int(kb % LF_STAGES);
      mbar_wait(&full[st], uint32_t((kb / LF_STAGES) & 1));
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sA + st * LF_A_TILE);
        const uint32_t b0 = smem_u32(sB + st * LF_B_TILE);
        // limb plane i of A against the N-concatenated planes B_0..B_{7-i}
        // (contiguous 16-feature chunks): column block j lands on diagonal
        // i + j, so each A plane is read once per k-block (12 MMAs, not 36)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint64_t ad = umma_desc(a0 + i * LF_A_PLANE, 128, 512);
#pragma unroll
          for (int n0 = 0; n0 < LF_BN * (8 - i); n0 += 256) {
            const int nn = LF_BN * (8 - i) - n0 < 256 ? LF_BN * (8 - i) - n0 : 256;
            const uint64_t bd = umma_desc(b0 + uint32_t(n0 / 16) * 512, 128, 512);
            mma_u8(tmem + uint32_t(i * LF_BN + n0), ad, bd, IDESC_M128 | (uint32_t(nn >> 3) << 17),
                   (kb == 0 && i == 0) ? 0u : 1u);
          }
        }
        mma_commit(&empty[st]);
      }
      __syncwarp();
    }
    if (lane == 0) mma_commit(tfull);
    __syncwarp();
  } else if (warp < 4) {
    // ---------------- epilogue: TMEM lane m = feature (u, a) of x
    if (nkb > 0) {
      mbar_wait(tfull, 0);
      tc_fence_after();
      // every TMA load has been consumed: the raw stages are free for red1/red2
      red1[threadIdx.x] = 0;
      red1[threadIdx.x + 128] = 0;
      lf_named_sync(1, 128);
      const int m = warp * 32 + lane;
      const int u = m >> 6, a = m & 63;
      const u64 w2 = (u == 0 && half == 0) ? 1ull : (u == 1 && half == 1) ? 4ull : u64(-2ll);
      const bool to_h1 = u == 1 && half == 1;
      const uint32_t lane_base = tmem + (uint32_t(warp * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < LF_BN; c0 += 8) {
        uint32_t v[8][8];
#pragma unroll
        for (int s = 0; s < 8; ++s) tmem_ld8(lane_base + uint32_t(s * LF_BN + c0), v[s]);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          u64 P = 0;
#pragma unroll
          for (int s = 0; s < 8; ++s) P += u64(v[s][q]) << (8 * s);
          const int cidx = a + c0 + q;
          atomicAdd(reinterpret_cast<unsigned long long*>(red2 + cidx), (unsigned long long)(w2 * P));
          if (to_h1) atomicAdd(reinterpret_cast<unsigned long long*>(red1 + cidx), (unsigned long long)P);
        }
      }
      tc_fence_before();
      lf_named_sync(1, 128);
      const int t = threadIdx.x;
      if (t < 127) {
        atomicAdd(reinterpret_cast<unsigned long long*>(acc2 + t), (unsigned long long)red2[t]);
        if (half == 1) atomicAdd(reinterpret_cast<unsigned long long*>(acc1 + t), (unsigned long long)red1[t]);
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

static bool lf_term(LfTerm& T, const uint64_t* a, const uint64_t* b0, const uint64_t* b1, u64 c0, u64 c1,
                    int64_t rows) {
  const int64_t ceilp = (rows + 1) / 2, floorp = rows / 2;
  T.c0 = c0;
  T.c1 = c1;
  T.has_b1 = b1 != nullptr;
  // a pair-view map with no rows (rows == 1, odd half) is given one row and
  // is never read past its zero fill: clamp to >= 1 and let the converters'
  // pair bound / TMA zero fill handle it
  const int64_t fl = floorp > 0 ? floorp : 0;
  bool ok = make_rows_tmap(&T.a_lo, a, ceilp, 128, LF_BK, 128);
  ok = ok && (fl > 0 ? make_rows_tmap(&T.a_hi, a, fl, 128, LF_BK, 128) : make_rows_tmap(&T.a_hi, a, 1, 128, LF_BK, 64));
  ok = ok && make_rows_tmap(&T.b0[0], b0, ceilp, 128, LF_BK, 128);
  ok = ok && (fl > 0 ? make_rows_tmap(&T.b0[1], b0, fl, 128, LF_BK, 128) : make_rows_tmap(&T.b0[1], b0, 1, 128, LF_BK, 64));
  if (b1) {
    ok = ok && make_rows_tmap(&T.b1[0], b1, ceilp, 128, LF_BK, 128);
    ok = ok && (fl > 0 ? make_rows_tmap(&T.b1[1], b1, fl, 128, LF_BK, 128) : make_rows_tmap(&T.b1[1], b1, 1, 128, LF_BK, 64));
  } else {
    T.b1[0] = T.b0[0];
    T.b1[1] = T.b0[1];
  }
  return ok;
}

// Called by r3_vfy_level_fold for d == 64 (same contract).
int level_fold_tc(int role, const uint64_t* xa, const uint64_t* xb, const uint64_t* ya, const uint64_t* yb,
                  int64_t N, uint64_t* acc1, uint64_t* acc2, cudaStream_t s) {
  if (N <= 1) return -1;   // caller's CUDA-core path (a lone row has no odd half)
  LfArgs args{};
  const u64 M1 = ~0ull;  // -1
  bool ok;
  if (role == 0) {
    ok = lf_term(args.t[0], xa, ya, nullptr, 1, 0, N);
    args.nterms = 1;
  } else if (role == 1) {  // -(m_x s_y) - (s_x m_y)
    ok = lf_term(args.t[0], xa, yb, nullptr, M1, 0, N) && lf_term(args.t[1], xb, ya, nullptr, M1, 0, N);
    args.nterms = 2;
  } else {  // m_x (m_y - s_y) - s_x m_y
    ok = lf_term(args.t[0], xa, ya, yb, 1, M1, N) && lf_term(args.t[1], xb, ya, nullptr, M1, 0, N);
    args.nterms = 2;
  }
  if (!ok) {
    set_error("r3_vfy_level_fold(tc): cuTensorMapEncodeTiled failed");
    return R3_ERR_CUDA;
  }
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
  level_fold_tc_kernel<<<grid, LF_THREADS, LF_SMEM, s>>>(args, (u64*)acc1, (u64*)acc2);
  return check_launch("r3_vfy_level_fold(tc)");
}
