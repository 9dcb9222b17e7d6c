// Dense-level verification folds for d = 16 on the tensor cores, the leg
// terms of several simulated parties in one pass (honest joint sessions).
//
// For d = 64 (lf_tc.cu) one leg term fills the MMA: M = 128 features are the
// 64 coefficients of the even and of the odd row of a pair.  At d = 16 a
// term has only 32 such features, so up to four terms share one MMA: A's
// 128 features are [term t: even 16 | odd 16] for t < 4 and B (one item per
// y half) holds the y features of terms {2h, 2h+1}.  The product X^T Y then
// contains every (term, term') block; the epilogue keeps the blocks with
// term = term' (a quarter of the MMA work -- still several times the u64
// throughput of the CUDA-core fold) and folds them exactly as lf_tc does:
//   h(1)[c] = sum_{a+b=c} P_oo[a][b],   h(2)[c] = sum_{a+b=c} (4 P_oo - 2 P_oe - 2 P_eo + P_ee)[a][b]
// accumulated into the output pair of the term's party.  The MMA, limb
// layout and pipeline are lf_tc's (12 N-concatenated kind::i8 MMAs per
// 32-pair K-step, K chunks <= 16384 pairs so the low diagonals are exact).
#include "tc_common.cuh"

namespace r3 {

constexpr int L16_BK = 32;                        // pairs per K-step
constexpr int L16_A_PLANE = 128 * L16_BK;         // 4 KB
constexpr int L16_B_PLANE = 64 * L16_BK;          // 2 KB
constexpr int L16_A_TILE = 8 * L16_A_PLANE;       // 32 KB
constexpr int L16_B_TILE = 8 * L16_B_PLANE;       // 16 KB
constexpr int L16_BOX = 16 * 8 * L16_BK;          // 16 u64 x 32 pairs = 4 KB
constexpr int L16_RAW = 16 * L16_BOX;             // A 8 boxes + B0 4 + B1 4 = 64 KB
constexpr int L16_STAGES = 2;
constexpr int L16_CONV = 12 * 32;                 // 256 A tasks + 128 B tasks per K-step
constexpr int L16_THREADS = 4 * 32 + L16_CONV + 2 * 32;
constexpr int L16_OFF_LIMB = L16_STAGES * L16_RAW;
constexpr int L16_OFF_BAR = L16_OFF_LIMB + L16_STAGES * (L16_A_TILE + L16_B_TILE);
constexpr int L16_SMEM = L16_OFF_BAR + 256 + 1024;
constexpr int64_t L16_MAX_K = 16384;

// One leg term: x, and y' = c0 y0 + c1 y1, each in the pair view (row p =
// component rows 2p, 2p+1: 32 u64).  *_lo maps cover ceil(N/2) pairs (the
// even row), *_hi maps floor(N/2) pairs (the odd row; a missing last odd
// row is the TMA zero fill).
struct L16Term {
  CUtensorMap x_lo, x_hi, y0_lo, y0_hi, y1_lo, y1_hi;
  u64 c0, c1;
  int has_y1, party;
};

struct L16Args {
  L16Term t[4];
  int nterms;
  int64_t npairs, kc, nchunks;
  u64* acc1[3];
  u64* acc2[3];
};

__device__ __forceinline__ void l16_named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void l16_read_row(const uint8_t* row, int sw, u64 (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(row + ((q ^ sw) << 4));
    v[2 * q] = x.x;
    v[2 * q + 1] = x.y;
  }
}


__global__ void __launch_bounds__(L16_THREADS, 1)
level_fold16_tc_kernel(const __grid_constant__ L16Args args) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself (keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sRaw = smem;
  uint8_t* sA = smem + L16_OFF_LIMB;
  uint8_t* sB = sA + L16_STAGES * L16_A_TILE;
  u64* red = reinterpret_cast<u64*>(smem);          // epilogue only: [party][h1 31 | h2 31]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L16_OFF_BAR);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = bars + L16_STAGES;
  uint64_t* full = bars + 2 * L16_STAGES;
  uint64_t* empty = bars + 3 * L16_STAGES;
  uint64_t* tfull = bars + 4 * L16_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int64_t item = blockIdx.x;
  const int ipc = args.nterms > 2 ? 2 : 1;          // items per chunk: y halves that hold terms
  const int half = int(item % ipc);                 // y terms {2 half, 2 half + 1}
  const int64_t chunk = item / ipc;
  const int64_t p0 = chunk * args.kc;
  const int64_t p1 = min(args.npairs, p0 + args.kc);
  const int64_t nkb = (p1 - p0 + L16_BK - 1) / L16_BK;
  const int nt = args.nterms;

  if (threadIdx.x == 0) {
    for (int s = 0; s < L16_STAGES; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], L16_CONV);
      mbar_init(&full[s], L16_CONV);
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
    // ---------------- TMA producer: slot c < 8: x of term c/2 (even / odd
    // row); 8 + c: y0 of term 2 half + c/2; 12 + c: y1 of that term
    if (lane == 0) {
      uint32_t bytes = 0;
      for (int c = 0; c < 8; ++c) bytes += (c >> 1) < nt ? L16_BOX : 0;
      for (int c = 0; c < 4; ++c) {
        const int tb = 2 * half + (c >> 1);
        if (tb < nt) bytes += L16_BOX * (args.t[tb].has_y1 ? 2 : 1);
      }
      for (int64_t kb = 0; kb < nkb; ++kb) {
        const int st = int(kb % L16_STAGES);
        if (kb >= L16_STAGES) mbar_wait(&raw_empty[st], uint32_t((kb / L16_STAGES - 1) & 1));
        const int y = int(p0 + kb * L16_BK);
        uint8_t* dst = sRaw + st * L16_RAW;
        mbar_expect_tx(&raw_full[st], bytes);
        for (int c = 0; c < 8; ++c) {
          const int t = c >> 1;
          if (t < nt) tma_load_2d(dst + c * L16_BOX, (c & 1) ? &args.t[t].x_hi : &args.t[t].x_lo, (c & 1) * 16, y,
                                  &raw_full[st]);
        }
        for (int c = 0; c < 4; ++c) {
          const int tb = 2 * half + (c >> 1);
          if (tb >= nt) continue;
          const L16Term& T = args.t[tb];
          tma_load_2d(dst + (8 + c) * L16_BOX, (c & 1) ? &T.y0_hi : &T.y0_lo, (c & 1) * 16, y, &raw_full[st]);
          if (T.has_y1)
            tma_load_2d(dst + (12 + c) * L16_BOX, (c & 1) ? &T.y1_hi : &T.y1_lo, (c & 1) * 16, y, &raw_full[st]);
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 16) {
    // ---------------- converters: thread = (pair row k, 16-feature chunk c)
    const int lt = threadIdx.x - 128;
    const bool isA = lt < 256;
    const int k = lt & 31;
    const int c = isA ? (lt >> 5) : ((lt - 256) >> 5);
    const int term = isA ? (c >> 1) : 2 * half + (c >> 1);
    const bool live_term = term < nt;
    const int sw = k & 7;
    for (int64_t kb = 0; kb < nkb; ++kb) {
      const int st = int(kb % L16_STAGES);
      mbar_wait(&raw_full[st], uint32_t((kb / L16_STAGES) & 1));
      const bool ok = live_term && p0 + kb * L16_BK + k < p1;   // pairs of the next chunk read as zero
      const uint8_t* raw = sRaw + st * L16_RAW;
      u64 v[16];
      if (ok) {
        if (isA) {
          l16_read_row(raw + c * L16_BOX + k * 128, sw, v);
        } else {
          const L16Term& T = args.t[term];
          l16_read_row(raw + (8 + c) * L16_BOX + k * 128, sw, v);
#pragma unroll
          for (int q = 0; q < 16; ++q) v[q] *= T.c0;
          if (T.has_y1) {
            u64 w[16];
            l16_read_row(raw + (12 + c) * L16_BOX + k * 128, sw, w);
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] += T.c1 * w[q];
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = 0;
      }
      fence_async_smem();   // generic-proxy reads before the next TMA write (WAR)
      mbar_arrive(&raw_empty[st]);
      uint4 pk[8];
      split_limbs16(v, pk);
      if (kb >= L16_STAGES) mbar_wait(&empty[st], uint32_t((kb / L16_STAGES - 1) & 1));
      // MN-major no-swizzle core layout: chunk stride 512 B, k-row stride 16 B
      uint8_t* dst = isA ? sA + st * L16_A_TILE : sB + st * L16_B_TILE;
      const int plane = isA ? L16_A_PLANE : L16_B_PLANE;
      const uint32_t off = uint32_t(c * 512 + k * 16);
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(dst + i * plane + off) = pk[i];
      fence_async_smem();
      mbar_arrive(&full[st]);
    }
  } else if (warp == 4 + 12 + 1) {
    // ---------------- MMA issuer (lf_tc's: 12 N-concatenated limb MMAs per K-step)
    constexpr uint32_t IDESC_M128 = idesc_u8(128, 0) | (1u << 15) | (1u << 16);   // A, B MN-major
    for (int64_t kb = 0; kb < nkb; ++kb) {
      const int st = int(kb % L16_STAGES);
      mbar_wait(&full[st], uint32_t((kb / L16_STAGES) & 1));
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sA + st * L16_A_TILE);
        const uint32_t b0 = smem_u32(sB + st * L16_B_TILE);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint64_t ad = umma_desc(a0 + i * L16_A_PLANE, 128, 512);
#pragma unroll
          for (int n0 = 0; n0 < 64 * (8 - i); n0 += 256) {
            const int nn = 64 * (8 - i) - n0 < 256 ? 64 * (8 - i) - n0 : 256;
            const uint64_t bd = umma_desc(b0 + uint32_t(n0 / 16) * 512, 128, 512);
            mma_u8(tmem + uint32_t(i * 64 + n0), ad, bd, IDESC_M128 | (uint32_t(nn >> 3) << 17),
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
    // ---------------- epilogue: warp w = TMEM lane quadrant w = A term w
    if (nkb > 0) {
      mbar_wait(tfull, 0);
      tc_fence_after();
      // every TMA load has been consumed: the raw stages are free for red
      for (int i = threadIdx.x; i < 3 * 64; i += 128) red[i] = 0;
      l16_named_sync(1, 128);
      const int t = warp;                                 // this lane's term
      const bool mine = t < nt && (t >> 1) == half;       // its y block is in this item
      if (mine) {
        const int u = lane >> 4, a = lane & 15;           // parity (0 even, 1 odd), coefficient
        const int p = args.t[t].party;
        u64* r1 = red + p * 64;
        u64* r2 = r1 + 31;
        const uint32_t lane_base = tmem + (uint32_t(warp * 32) << 16) + uint32_t(32 * (t & 1));
#pragma unroll 1
        for (int c0 = 0; c0 < 32; c0 += 8) {
          uint32_t v[8][8];
#pragma unroll
          for (int s = 0; s < 8; ++s) tmem_ld8(lane_base + uint32_t(s * 64 + c0), v[s]);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int n = c0 + q, vpar = n >> 4, b = n & 15;
            const u64 P = recombine8(v[0][q], v[1][q], v[2][q], v[3][q], v[4][q], v[5][q], v[6][q], v[7][q]);
            const u64 w2 = (u & vpar) ? 4ull : (u | vpar) ? u64(-2ll) : 1ull;
            atomicAdd(reinterpret_cast<unsigned long long*>(r2 + a + b), (unsigned long long)(w2 * P));
            if (u & vpar) atomicAdd(reinterpret_cast<unsigned long long*>(r1 + a + b), (unsigned long long)P);
          }
        }
      }
      tc_fence_before();
      l16_named_sync(1, 128);
      for (int i = threadIdx.x; i < 3 * 62; i += 128) {
        const int p = i / 62, j = i % 62;
        if (!args.acc1[p]) continue;
        const u64 val = red[p * 64 + j];
        if (j < 31) atomicAdd(reinterpret_cast<unsigned long long*>(args.acc1[p] + j), (unsigned long long)val);
        else atomicAdd(reinterpret_cast<unsigned long long*>(args.acc2[p] + (j - 31)), (unsigned long long)val);
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

static bool l16_pair_maps(CUtensorMap* lo, CUtensorMap* hi, const uint64_t* a, int64_t rows) {
  const int64_t ceilp = (rows + 1) / 2, floorp = rows / 2;
  bool ok = make_rows_tmap(lo, a, ceilp, 32, L16_BK, 32);
  // no odd rows at all (rows == 1): a one-row map, never read past the pair bound
  ok = ok && make_rows_tmap(hi, a, floorp > 0 ? floorp : 1, 32, L16_BK, 32);
  return ok;
}

// Leg-term folds of up to four terms (d = 16) in one pass; term k belongs to
// party party[k] and adds its h(1)/h(2) into acc1[party] / acc2[party]
// (2 d - 1 = 31 unreduced words each, zeroed here).  x / y0 / y1 are (N, 16)
// row-major component arrays; y' = c0 y0 + c1 y1 (y1 may be null).
extern "C" int r3_vfy_level_fold16_tc(int nterms, const int* party, const uint64_t* const* xs,
                                      const uint64_t* const* y0s, const uint64_t* const* y1s, const int64_t* c0,
                                      const int64_t* c1, int64_t N, uint64_t* const* acc1, uint64_t* const* acc2,
                                      void* stream) {
  if (nterms < 1 || nterms > 4 || !party || !xs || !y0s || !c0 || !acc1 || !acc2 || N < 2 ||
      N > (int64_t(1) << 32)) {
    set_error("r3_vfy_level_fold16_tc: bad arguments (1..4 terms, N >= 2)");
    return R3_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  L16Args args{};
  for (int p = 0; p < 3; ++p) {
    args.acc1[p] = reinterpret_cast<u64*>(acc1[p]);
    args.acc2[p] = reinterpret_cast<u64*>(acc2[p]);
    if ((acc1[p] != nullptr) != (acc2[p] != nullptr)) {
      set_error("r3_vfy_level_fold16_tc: acc1/acc2 must be given together");
      return R3_ERR_ARG;
    }
    if (acc1[p] && (cudaMemsetAsync(acc1[p], 0, 31 * 8, s) != cudaSuccess ||
                    cudaMemsetAsync(acc2[p], 0, 31 * 8, s) != cudaSuccess)) {
      set_error("r3_vfy_level_fold16_tc: memset failed");
      return R3_ERR_CUDA;
    }
  }
  bool ok = true;
  for (int k = 0; k < nterms; ++k) {
    L16Term& T = args.t[k];
    if (party[k] < 0 || party[k] > 2 || !acc1[party[k]] || !xs[k] || !y0s[k] ||
        ((uintptr_t(xs[k]) | uintptr_t(y0s[k]) | uintptr_t(y1s ? y1s[k] : nullptr)) & 15)) {
      set_error("r3_vfy_level_fold16_tc: bad term %d", k);
      return R3_ERR_ARG;
    }
    T.party = party[k];
    T.c0 = u64(c0[k]);
    T.c1 = c1 ? u64(c1[k]) : 0ull;
    T.has_y1 = (y1s && y1s[k]) ? 1 : 0;
    ok = ok && l16_pair_maps(&T.x_lo, &T.x_hi, xs[k], N) && l16_pair_maps(&T.y0_lo, &T.y0_hi, y0s[k], N);
    if (T.has_y1) ok = ok && l16_pair_maps(&T.y1_lo, &T.y1_hi, y1s[k], N);
    else {
      T.y1_lo = T.y0_lo;
      T.y1_hi = T.y0_hi;
    }
  }
  if (!ok) {
    set_error("r3_vfy_level_fold16_tc: cuTensorMapEncodeTiled failed");
    return R3_ERR_CUDA;
  }
  args.nterms = nterms;
  args.npairs = (N + 1) / 2;
  int64_t nchunks = (args.npairs + L16_MAX_K - 1) / L16_MAX_K;
  const int64_t items_per_chunk = nterms > 2 ? 2 : 1;
  const int64_t waves = (nchunks * items_per_chunk + num_sms() - 1) / num_sms();
  int64_t want = waves * num_sms() / items_per_chunk;   // fill the last wave
  const int64_t min_kc = 8 * L16_BK;
  if (want * min_kc > args.npairs) want = (args.npairs + min_kc - 1) / min_kc;
  if (want > nchunks) nchunks = want;
  int64_t kc = (args.npairs + nchunks - 1) / nchunks;
  kc = (kc + L16_BK - 1) / L16_BK * L16_BK;
  nchunks = (args.npairs + kc - 1) / kc;
  args.kc = kc;
  args.nchunks = nchunks;
  ensure_smem(level_fold16_tc_kernel, L16_SMEM);
  level_fold16_tc_kernel<<<unsigned(nchunks * items_per_chunk), L16_THREADS, L16_SMEM, s>>>(args);
  return check_launch("r3_vfy_level_fold16_tc");
}
