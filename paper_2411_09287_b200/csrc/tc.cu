// tcgen05 (5th-gen tensor core) kernels: exact mod-2^64 GEMMs on byte limbs.
//
// A u64 value is 8 little-endian byte limbs, a = sum_i a_i 2^(8i).  Mod 2^64
// only the limb products with i + j <= 7 survive:
//     A . B  =  sum_{s=0..7} 2^(8s) D_s,   D_s = sum_{i+j=s} A_i . B_j
// so one u64 GEMM is 36 u8 x u8 -> s32 GEMMs (tcgen05.mma kind::i8), grouped
// into 8 TMEM accumulators (one per diagonal s).  Every D_s is exact: with
// K <= 8192 its true value is < (s+1) K 255^2 < 2^32, so the unsigned 32-bit
// accumulator holds it without wrap, and the epilogue recombines the 8
// diagonals in u64 (SURVEY.md "hard part" 6).
//
// r3_gr_matmul2_tc: out[r] = P0[r] . M0 (+ P1[r] . M1) for GR(2^64, 64) rows
// -- the "many elements times one public element" contraction of the
// verification (line evaluations f0 (1 - zeta) + f1 zeta, power tables).
// M = 64 x 64, so K = N = 64: per 128-row tile and operand 72 MMAs of
// 128 x 64 x 32 into 8 x 64 TMEM columns (the full 512-column TMEM).
//
// smem operands use the canonical K-major no-swizzle layout: 8-row x 16-byte
// core matrices, core (g, kc) at (kc * G + g) * 128 bytes (G = rows / 8), so
// the descriptor's SBO = 128 B (next 8 rows) and LBO = G * 128 B (next 16 K).
#include "tc_common.cuh"

namespace r3 {
constexpr int TC_ROWS = 128;        // MMA M
constexpr int TC_D = 64;            // GR degree = K = N
constexpr int A_PLANE = TC_ROWS * TC_D;   // bytes per limb plane of A (8 KB)
constexpr int B_PLANE = TC_D * TC_D;      // bytes per limb plane of B (4 KB)

// ---------------------------------------------------------------------------
// Warp-specialised pipelined form: out = P0 . M0 (+ P1 . M1)
//   warps 0-3   epilogue: TMEM diagonals -> u64 recombination -> global
//   warps 4-11  loaders : 16 consecutive u64 of a row -> 8 limb planes (smem)
//   warp 12     MMA issue (one elected lane)
// Two operand stages (one per operand of a tile, or consecutive tiles) are
// ping-ponged through mbarriers; the 512 TMEM columns hold the 8 diagonal
// accumulators of one 128 x 64 tile.
// ---------------------------------------------------------------------------
constexpr int W_EPI = 4, W_LOAD = 8;
constexpr int WS_THREADS = (W_EPI + W_LOAD + 1) * 32;
constexpr int STAGE_BYTES = 8 * A_PLANE;                 // 64 KB: one operand tile in limbs
constexpr int WS_SMEM = 2 * STAGE_BYTES + 2 * 8 * B_PLANE + 128;

struct RowOperand {
  const u64* p;
  int64_t rs;
  int64_t nvalid;
};


__global__ void __launch_bounds__(WS_THREADS, 1)
gr_matmul2_tc_kernel(RowOperand P0, RowOperand P1, int nops, const u64* __restrict__ M0,
                     const u64* __restrict__ M1, u64* __restrict__ out, int64_t rows, u64 mask) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA[2] = {smem, smem + STAGE_BYTES};
  uint8_t* sB[2] = {smem + 2 * STAGE_BYTES, smem + 2 * STAGE_BYTES + 8 * B_PLANE};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGE_BYTES + 16 * B_PLANE);
  uint64_t* full = bars;        // [2] loaders -> MMA
  uint64_t* empty = bars + 2;   // [2] MMA -> loaders
  uint64_t* tfull = bars + 4;   // MMA -> epilogue
  uint64_t* tempty = bars + 5;  // epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // B operands: B_j[n][k] = limb j of M[k][n]
  for (int op = 0; op < nops; ++op) {
    const u64* M = op ? M1 : M0;
    for (int e = tid; e < TC_D * TC_D; e += WS_THREADS) {
      const int k = e / TC_D, n = e % TC_D;
      const u64 v = M[e];
#pragma unroll
      for (int j = 0; j < 8; ++j) sB[op][j * B_PLANE + core_off(n, k, TC_D / 8)] = uint8_t(v >> (8 * j));
    }
  }
  if (tid == 0) {
    mbar_init(&full[0], W_LOAD * 32);
    mbar_init(&full[1], W_LOAD * 32);
    mbar_init(&empty[0], 1);
    mbar_init(&empty[1], 1);
    mbar_init(tfull, 1);
    mbar_init(tempty, W_EPI * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (rows + TC_ROWS - 1) / TC_ROWS;

  if (warp >= W_EPI && warp < W_EPI + W_LOAD) {
    // ------------------------------ loaders
    // Flat stream of units (tile, operand, half): the loads of unit u+1 are in
    // flight while unit u is split into limb planes (register double buffer).
    const int ltid = tid - W_EPI * 32;
    const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int64_t nunits = my_tiles * nops * 2;
    uint32_t w[2][32];
    auto load_unit = [&](int64_t u, uint32_t (&dst)[32]) {
      const int64_t t = blockIdx.x + (u / (2 * nops)) * gridDim.x;
      const int op = int((u >> 1) % nops), h = int(u & 1);
      const RowOperand P = op ? P1 : P0;
      const int task = ltid + h * W_LOAD * 32;
      const int r = task & (TC_ROWS - 1), k0 = (task >> 7) * 16;
      const int64_t row = t * TC_ROWS + r;
      if (row < rows && row < P.nvalid) {
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(P.p + row * P.rs + k0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          ulonglong2 v = __ldg(src + q);
          dst[4 * q + 0] = uint32_t(v.x);
          dst[4 * q + 1] = uint32_t(v.x >> 32);
          dst[4 * q + 2] = uint32_t(v.y);
          dst[4 * q + 3] = uint32_t(v.y >> 32);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) dst[q] = 0;
      }
    };
    int stage = 0;
    uint32_t ephase0 = 0, ephase1 = 0;
    int used0 = 0, used1 = 0;
    // a unit with h == 0 opens a stage, h == 1 closes it; units come in pairs
    auto process = [&](int h, const uint32_t (&x)[32]) {
      if (h == 0) {
        if (stage == 0) {
          if (used0) { mbar_wait(&empty[0], ephase0); ephase0 ^= 1; }
          used0 = 1;
        } else {
          if (used1) { mbar_wait(&empty[1], ephase1); ephase1 ^= 1; }
          used1 = 1;
        }
      }
      const int task = ltid + h * W_LOAD * 32;
      const int r = task & (TC_ROWS - 1), k0 = (task >> 7) * 16;
      uint8_t* dst = (stage ? sA[1] : sA[0]) + core_off(r, k0, TC_ROWS / 8);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int hiw = i >> 2, bi = i & 3;
        uint4 pk;
        pk.x = gather_byte(x[0 + hiw], x[2 + hiw], x[4 + hiw], x[6 + hiw], bi);
        pk.y = gather_byte(x[8 + hiw], x[10 + hiw], x[12 + hiw], x[14 + hiw], bi);
        pk.z = gather_byte(x[16 + hiw], x[18 + hiw], x[20 + hiw], x[22 + hiw], bi);
        pk.w = gather_byte(x[24 + hiw], x[26 + hiw], x[28 + hiw], x[30 + hiw], bi);
        *reinterpret_cast<uint4*>(dst + i * A_PLANE) = pk;
      }
      if (h == 1) {
        fence_async_smem();
        mbar_arrive(&full[stage]);
        stage ^= 1;
      }
    };
    if (nunits > 0) load_unit(0, w[0]);
#pragma unroll 1
    for (int64_t u = 0; u < nunits; u += 2) {
      load_unit(u + 1, w[1]);                     // nunits is even
      process(0, w[0]);
      if (u + 2 < nunits) load_unit(u + 2, w[0]);
      process(1, w[1]);
    }
  } else if (warp == W_EPI + W_LOAD) {
    // ------------------------------ MMA issuer
    constexpr uint32_t IDESC = idesc_u8(TC_ROWS, TC_D);
    int stage = 0;
    uint32_t fphase[2] = {0, 0};
    uint32_t tphase = 0;
    bool first_tile = true;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      if (!first_tile) {
        mbar_wait(tempty, tphase);
        tphase ^= 1;
      }
      first_tile = false;
      tc_fence_after();
      for (int op = 0; op < nops; ++op) {
        mbar_wait(&full[stage], fphase[stage]);
        fphase[stage] ^= 1;
        tc_fence_after();
        if (lane == 0) {
#pragma unroll 1
          for (int s = 0; s < 8; ++s) {
            const uint32_t d_tmem = tmem + uint32_t(s * TC_D);
            for (int i = 0; i <= s; ++i) {
              const int j = s - i;
              for (int kk = 0; kk < TC_D; kk += 32) {
                const uint32_t a_addr = smem_u32(sA[stage] + i * A_PLANE) + uint32_t((kk >> 4) * (TC_ROWS / 8) * 128);
                const uint32_t b_addr = smem_u32(sB[op] + j * B_PLANE) + uint32_t((kk >> 4) * (TC_D / 8) * 128);
                const uint64_t ad = umma_desc(a_addr, (TC_ROWS / 8) * 128, 128);
                const uint64_t bd = umma_desc(b_addr, (TC_D / 8) * 128, 128);
                const bool acc = op > 0 || i > 0 || kk > 0;
                mma_u8(d_tmem, ad, bd, IDESC, acc ? 1u : 0u);
              }
            }
          }
          mma_commit(&empty[stage]);
          if (op == nops - 1) mma_commit(tfull);
        }
        __syncwarp();
        stage ^= 1;
      }
    }
  } else if (warp < W_EPI) {
    // ------------------------------ epilogue: warp e reads TMEM lane quadrant
    // e % 4 (rows) and column half e / 4; 8 columns x 8 diagonals per batch
    uint32_t phase = 0;
    const int quad = warp & 3;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      mbar_wait(tfull, phase);
      phase ^= 1;
      tc_fence_after();
      const int64_t row = t * TC_ROWS + quad * 32 + lane;
      const uint32_t lane_base = tmem + (uint32_t(quad * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < TC_D; c0 += 8) {
        uint32_t v[8][8];
#pragma unroll
        for (int s = 0; s < 8; ++s) tmem_ld8(lane_base + uint32_t(s * TC_D + c0), v[s]);
        tmem_wait_ld();
        u64 acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          u64 a = 0;
#pragma unroll
          for (int s = 0; s < 8; ++s) a += u64(v[s][q]) << (8 * s);
          acc[q] = a & mask;
        }
        if (row < rows) {
          ulonglong2* o = reinterpret_cast<ulonglong2*>(out + row * TC_D + c0);
#pragma unroll
          for (int q = 0; q < 8; q += 2) o[q >> 1] = make_ulonglong2(acc[q], acc[q + 1]);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace r3

using namespace r3;

extern "C" int r3_gr_matmul2_tc(const uint64_t* p0, int64_t rs0, int64_t nv0, const uint64_t* p1, int64_t rs1,
                                int64_t nv1, const uint64_t* M0, const uint64_t* M1, uint64_t* out, int64_t rows,
                                uint64_t mask, void* stream) {
  if (!p0 || !M0 || rows < 0 || ((rs0 | rs1) & 1) || ((uintptr_t(p0) | uintptr_t(p1)) & 15)) {
    set_error("r3_gr_matmul2_tc: bad arguments (need 16-byte aligned rows)");
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gr_matmul2_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WS_SMEM);
    attr = true;
  }
  RowOperand a{reinterpret_cast<const u64*>(p0), rs0, nv0};
  RowOperand b{reinterpret_cast<const u64*>(p1), rs1, nv1};
  const int nops = p1 ? 2 : 1;
  const int64_t tiles = (rows + TC_ROWS - 1) / TC_ROWS;
  const unsigned grid = unsigned(tiles < kNumSMs ? tiles : kNumSMs);
  gr_matmul2_tc_kernel<<<grid, WS_THREADS, WS_SMEM, as_stream(stream)>>>(a, b, nops, (const u64*)M0,
                                                                          (const u64*)M1, (u64*)out, rows, mask);
  return check_launch("r3_gr_matmul2_tc");
}
