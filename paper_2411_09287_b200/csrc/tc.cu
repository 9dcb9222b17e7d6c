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
// M = 64 x 64, so K = N = 64: per 128-row tile, operand and output-column
// half 16 MMAs (the 36 limb products of both K-halves, N-concatenated) into
// 8 x 32 TMEM columns; the two halves double-buffer the 512-column TMEM.
//
// smem operands use the canonical K-major no-swizzle layout: 8-row x 16-byte
// core matrices, core (g, kc) at (kc * G + g) * 128 bytes (G = rows / 8), so
// the descriptor's SBO = 128 B (next 8 rows) and LBO = G * 128 B (next 16 K).
#include "tc_common.cuh"

namespace r3 {
constexpr int TC_ROWS = 128;        // MMA M
constexpr int TC_D = 64;            // GR degree = K = N of one limb product
constexpr int TC_KH = 32;           // K per unit (one MMA K-step of kind::i8)

// ---------------------------------------------------------------------------
// out = P0 . M0 (+ P1 . M1).  A unit is (tile of 128 rows, operand, K-half):
// 128 x 32 u64 = 32 KB of HBM, moved by two TMA tile loads (16 u64 x 128
// rows each, 128-byte swizzle so the converters read it bank-conflict
// free), split into 8 byte-limb planes (128 x 32 B, K-major no-swizzle core
// matrices) by the converter warps, and consumed by MMAs that multiply limb
// plane i of A by the N-concatenated limb planes [B_0 .. B_{7-i}] of the
// public matrix, whose column block j lands on diagonal i + j of the TMEM
// accumulator.  Each A plane is read by the tensor core once per unit and
// output half instead of once per (i, j) limb product.
// ---------------------------------------------------------------------------
// eight epilogue warps: two per TMEM lane quadrant, each recombining half
// of a piece's columns (four warps left the tensor pipe ~34 % active in the
// table build: the epilogue, not the MMA, paced the TMEM double buffer)
constexpr int W_EPI = 8, W_CONV = 8;
constexpr int WS_THREADS = (W_EPI + W_CONV + 2) * 32;
constexpr int RAW_BYTES = TC_ROWS * TC_KH * 8;           // 32 KB
constexpr int LIMB_PLANE = TC_ROWS * TC_KH;              // 4 KB
constexpr int BALL_ROWS = 8 * TC_D;                      // 512 = 8 limb planes of N
constexpr int BALL_BYTES = BALL_ROWS * TC_D;             // 32 KB per operand

// ---------------------------------------------------------------------------
// Double-buffered TMEM.  The accumulators of a 128 x 64 output tile would
// fill all 512 TMEM columns, so the epilogue (bound by TMEM reads: 256 KB
// per tile) and the next tile's MMAs would run one after the other.  A tile
// is computed as two column halves (output columns 32 h .. 32 h + 31),
// each with its own 256-column accumulator (diagonal s at 256 h + 32 s): the
// epilogue drains half 0 while the MMAs of half 1 run, and half 1 while the
// next tile's half 0 runs.  Both halves read the same limb planes, so a
// tile's units stay resident until its half-1 MMAs: each stage is converted
// IN PLACE (raw rows -> registers, converter barrier, limb planes written
// over the raw bytes), which gives 5 stages of 32 KB in the shared memory
// the raw + limb stages used before, and a stage is released unit by unit
// as half 1 consumes it, so the next tile's loads start early.
// B_all rows are ordered n' = 256 h + 32 j + (n mod 32) (half h, limb j) so
// one half's N-concatenated limb planes are contiguous: 8 MMAs of
// N = 32 (8 - i) per unit and half.
//   warps 0-3   epilogue       warps 4-11  converters
//   warp 12     TMA producer   warp 13     MMA issuer
// ---------------------------------------------------------------------------
constexpr int DB_STAGES = 5;
constexpr int DB_OFF_B = DB_STAGES * RAW_BYTES;
constexpr int DB_OFF_BAR = DB_OFF_B + 2 * BALL_BYTES;
constexpr int DB_SMEM = DB_OFF_BAR + 256 + 1024;
constexpr int DB_HALF = TC_D / 2;                        // output columns per half

__device__ __forceinline__ void conv_named_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(W_CONV * 32) : "memory");
}

// Jobs of one launch: every job is rows of P0 (and P1) times the same
// public M0 (M1), so one CTA's B planes serve all of them (the line
// evaluations of all components of a reduction level share M(1 - z), M(z));
// tiles are numbered job after job (tile0 = prefix sums).
constexpr int MM2_MAX_JOBS = 8;
struct Mm2Jobs {
  CUtensorMap tm[MM2_MAX_JOBS][2];
  u64* out[MM2_MAX_JOBS];
  int64_t rows[MM2_MAX_JOBS];
  int64_t tile0[MM2_MAX_JOBS + 1];
  int njobs, nops;
};

__device__ __forceinline__ int mm2_job(const Mm2Jobs& J, int64_t t) {
  int j = 0;
#pragma unroll 1
  while (j + 1 < J.njobs && t >= J.tile0[j + 1]) ++j;
  return j;
}

// ---------------------------------------------------------------------------
// Epilogue of one warp's share of a half tile: four blocks of 16 TMEM lanes x
// 8 columns (it = it0 .. it0 + 3), each 8 limb diagonals recombined into
// u64 words.  Software-pipelined: the TMEM reads of block k + 1 are in
// flight while block k is recombined and stored, so the tcgen05.ld latency
// is paid once per half instead of once per block.  (tcgen05.wait::ld waits
// for every outstanding load, so the next block's loads are issued after
// the wait of the current one; the empty asm pins keep every use of a
// buffer after its wait.)
// ---------------------------------------------------------------------------
#ifndef R3_EPI_PIPE
#define R3_EPI_PIPE 1
#endif
__device__ __forceinline__ void tmem_ld_diag8(uint32_t taddr, uint32_t (&v)[8][4]) {
#pragma unroll
  for (int s = 0; s < 8; ++s) tmem_ld_16x256(taddr + uint32_t(DB_HALF * s), v[s]);
}
__device__ __forceinline__ void tmem_pin8(uint32_t (&v)[8][4]) {
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q) asm volatile("" : "+r"(v[s][q]));
}
__device__ __forceinline__ void epi_store_block(const uint32_t (&v)[8][4], u64 mask, u64* __restrict__ out,
                                                int64_t row, int64_t rows, int col) {
  u64 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    acc[q] = recombine8(v[0][q], v[1][q], v[2][q], v[3][q], v[4][q], v[5][q], v[6][q], v[7][q]) & mask;
  if (row < rows) *reinterpret_cast<ulonglong2*>(out + row * TC_D + col) = make_ulonglong2(acc[0], acc[1]);
  if (row + 8 < rows)
    *reinterpret_cast<ulonglong2*>(out + (row + 8) * TC_D + col) = make_ulonglong2(acc[2], acc[3]);
}
// tbase = TMEM address of (lane quadrant row 0, this accumulator buffer);
// row0 = the quadrant's first output row, col0 = the half's first column
__device__ __forceinline__ void epi_half(uint32_t tbase, int it0, u64 mask, u64* __restrict__ out, int64_t row0,
                                         int64_t rows, int col0, int rq, int cq) {
#define R3_TA(it) (tbase + (uint32_t(((it) & 1) * 16) << 16) + uint32_t(8 * ((it) >> 1)))
#define R3_ROW(it) (row0 + ((it) & 1) * 16 + rq)
#define R3_COL(it) (col0 + 8 * ((it) >> 1) + cq)
#if R3_EPI_PIPE
  uint32_t va[8][4], vb[8][4];
  tmem_ld_diag8(R3_TA(it0), va);
  tmem_wait_ld();
  tmem_pin8(va);
  tmem_ld_diag8(R3_TA(it0 + 1), vb);
  epi_store_block(va, mask, out, R3_ROW(it0), rows, R3_COL(it0));
  tmem_wait_ld();
  tmem_pin8(vb);
  tmem_ld_diag8(R3_TA(it0 + 2), va);
  epi_store_block(vb, mask, out, R3_ROW(it0 + 1), rows, R3_COL(it0 + 1));
  tmem_wait_ld();
  tmem_pin8(va);
  tmem_ld_diag8(R3_TA(it0 + 3), vb);
  epi_store_block(va, mask, out, R3_ROW(it0 + 2), rows, R3_COL(it0 + 2));
  tmem_wait_ld();
  tmem_pin8(vb);
  epi_store_block(vb, mask, out, R3_ROW(it0 + 3), rows, R3_COL(it0 + 3));
#else
#pragma unroll 1
  for (int it = it0; it < it0 + 4; ++it) {
    uint32_t v[8][4];
    tmem_ld_diag8(R3_TA(it), v);
    tmem_wait_ld();
    epi_store_block(v, mask, out, R3_ROW(it), rows, R3_COL(it));
  }
#endif
#undef R3_TA
#undef R3_ROW
#undef R3_COL
}
static_assert(DB_HALF / 8 == 4, "epi_half handles four 8-column blocks per warp");

__global__ void __launch_bounds__(WS_THREADS, 1)
gr_matmul2_db_kernel(const __grid_constant__ Mm2Jobs J, const u64* __restrict__ M0, const u64* __restrict__ M1,
                     u64 mask) {
  const int nops = J.nops;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself (keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sStage = smem;
  uint8_t* sB = smem + DB_OFF_B;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + DB_OFF_BAR);
  uint64_t* raw_full = bars;                       // [S] TMA -> converters
  uint64_t* limb_full = bars + DB_STAGES;          // [S] converters -> MMA
  uint64_t* empty = bars + 2 * DB_STAGES;          // [S] MMA (half 1) -> TMA
  uint64_t* tfull = bars + 3 * DB_STAGES;          // [2] MMA -> epilogue, per half
  uint64_t* tempty = tfull + 2;                    // [2] epilogue -> MMA, per half
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // B_all[op]: row 256 h + 32 j + c holds limb j of column 32 h + c of M
  for (int op = 0; op < nops; ++op) {
    const u64* M = op ? M1 : M0;
    uint8_t* dst = sB + op * BALL_BYTES;
    for (int e = tid; e < TC_D * TC_D; e += WS_THREADS) {
      const int k = e / TC_D, n = e % TC_D;
      const int h = n / DB_HALF, c = n % DB_HALF;
      const u64 v = M[e];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        dst[core_off(256 * h + DB_HALF * j + c, k, BALL_ROWS / 8)] = uint8_t(v >> (8 * j));
    }
  }
  if (tid == 0) {
    for (int i = 0; i < DB_STAGES; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&limb_full[i], W_CONV * 32);
      mbar_init(&empty[i], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&tfull[h], 1);
      mbar_init(&tempty[h], W_EPI * 32);
    }
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
  const int64_t ntiles = J.tile0[J.njobs];
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int upt = 2 * nops;                        // units per tile: (operand, K-half)
  const int64_t nunits = my_tiles * upt;

  if (warp == W_EPI + W_CONV) {
    // ------------------------------ TMA producer
    if (lane == 0) {
      for (int64_t g = 0; g < nunits; ++g) {
        const int st = int(g % DB_STAGES);
        if (g >= DB_STAGES) mbar_wait(&empty[st], uint32_t((g / DB_STAGES - 1) & 1));
        const int64_t t = blockIdx.x + (g / upt) * gridDim.x;
        const int j = mm2_job(J, t);
        const int64_t lt = t - J.tile0[j];
        const int op = int((g >> 1) % nops), h = int(g & 1);
        const CUtensorMap* map = &J.tm[j][op];
        uint8_t* dst = sStage + st * RAW_BYTES;
        mbar_expect_tx(&raw_full[st], RAW_BYTES);
        tma_load_2d(dst, map, h * TC_KH, int(lt * TC_ROWS), &raw_full[st]);
        tma_load_2d(dst + RAW_BYTES / 2, map, h * TC_KH + 16, int(lt * TC_ROWS), &raw_full[st]);
      }
    }
    __syncwarp();
  } else if (warp >= W_EPI && warp < W_EPI + W_CONV) {
    // ------------------------------ converters (in place): thread = (row r, box c)
    const int ct = tid - W_EPI * 32;
    const int r = ct & (TC_ROWS - 1), c = ct >> 7;
    const int sw = r & 7;
    for (int64_t g = 0; g < nunits; ++g) {
      const int st = int(g % DB_STAGES);
      mbar_wait(&raw_full[st], uint32_t((g / DB_STAGES) & 1));
      uint8_t* stage = sStage + st * RAW_BYTES;
      const uint8_t* src = stage + c * (RAW_BYTES / 2) + r * 128;
      uint32_t x[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + ((q ^ sw) << 4));
        x[4 * q + 0] = v.x;
        x[4 * q + 1] = v.y;
        x[4 * q + 2] = v.z;
        x[4 * q + 3] = v.w;
      }
      conv_named_sync();    // every raw row of the stage is in registers before any limb write
      uint8_t* dst = stage + core_off(r, c * 16, TC_ROWS / 8);
      uint4 pk[8];
      split_limbs16(x, pk);
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(dst + i * LIMB_PLANE) = pk[i];
      fence_async_smem();   // generic limb writes -> tensor-core (async proxy) reads
      mbar_arrive(&limb_full[st]);
    }
  } else if (warp == W_EPI + W_CONV + 1) {
    // ------------------------------ MMA issuer
    uint32_t tph[2] = {0, 0};
    for (int64_t g0 = 0; g0 < nunits; g0 += upt) {
      for (int h = 0; h < 2; ++h) {
        if (g0 > 0) {
          mbar_wait(&tempty[h], tph[h]);
          tph[h] ^= 1;
        }
        for (int uu = 0; uu < upt; ++uu) {
          const int64_t g = g0 + uu;
          const int st = int(g % DB_STAGES);
          const int op = uu >> 1, kh = uu & 1;
          if (h == 0) mbar_wait(&limb_full[st], uint32_t((g / DB_STAGES) & 1));
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a0 = smem_u32(sStage + st * RAW_BYTES);
            // K-half kh = core columns 2 kh, 2 kh + 1; half h = row groups 32 h ..
            const uint32_t b0 = smem_u32(sB + op * BALL_BYTES) +
                                uint32_t((2 * kh * (BALL_ROWS / 8) + 32 * h) * 128);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint64_t ad = umma_desc(a0 + i * LIMB_PLANE, (TC_ROWS / 8) * 128, 128);
              const uint64_t bd = umma_desc(b0, (BALL_ROWS / 8) * 128, 128);
              const bool acc = !(uu == 0 && i == 0);
              mma_u8(tmem + uint32_t(256 * h + DB_HALF * i), ad, bd, idesc_u8(TC_ROWS, DB_HALF * (8 - i)),
                     acc ? 1u : 0u);
            }
            if (h == 1) mma_commit(&empty[st]);
            if (uu == upt - 1) mma_commit(&tfull[h]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp < W_EPI) {
    // ------------------------------ epilogue: warp e reads TMEM lane quadrant e
    // (16-lane x 8-column loads: 4 threads per row, so every store writes
    // 8 rows x 64 contiguous bytes instead of 32 rows x 16 bytes)
    uint32_t ph[2] = {0, 0};
    const int quad = warp & 3, grp = warp >> 2;
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int j = mm2_job(J, t);
      const int64_t lt = t - J.tile0[j];
      const int64_t rows = J.rows[j];
      u64* __restrict__ out = J.out[j];
      for (int h = 0; h < 2; ++h) {
        mbar_wait(&tfull[h], ph[h]);
        ph[h] ^= 1;
        tc_fence_after();
        epi_half(tmem + (uint32_t(quad * 32) << 16) + uint32_t(256 * h), grp * (DB_HALF / 8), mask, out,
                 lt * TC_ROWS + quad * 32, rows, DB_HALF * h, rq, cq);
        tc_fence_before();
        mbar_arrive(&tempty[h]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// One operand, Q <= 4 public matrices: out_q[r] = P[r] . M_q (the four
// level-2 tables V_a = r^(4j) . C_a of one verification come from ONE pass
// over the r^(4j) table instead of four).  Same unit / in-place stage / TMEM
// double-buffering scheme as gr_matmul2_db_kernel; a tile's limb planes stay
// resident for its 2 Q pieces (matrix q, output-column half h), and the
// 4 x 32 KB of B planes leave room for 3 stages.
// ---------------------------------------------------------------------------
constexpr int MQ_MAX = 4;
// QM matrices resident, ST raw stages (a tile's two K-units stay in place
// until its last piece's MMA): four matrices leave room for 1.5 tiles of
// stages, two matrices for 2.5 (ncu r04u: the converters of the four-matrix
// form waited on TMA data for 38 % of the stall samples)
template <int QM>
struct MqLayout {
  static constexpr int ST = QM == 4 ? 3 : 5;
  static constexpr int OFF_B = ST * RAW_BYTES;
  static constexpr int OFF_BAR = OFF_B + QM * BALL_BYTES;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
};
static_assert(MqLayout<4>::SMEM <= 232448 && MqLayout<2>::SMEM <= 232448, "gr_matmul_q shared memory");

struct MqArgs {
  const u64* M[MQ_MAX];
  u64* out[MQ_MAX];
  int q;
  int k16;   // 1: P rows hold 16 words and each M is 16 x 64 (K = 16: one
             // K-unit per tile, the unit's upper 16 K columns meet zero rows of B)
};

template <int QM>
__global__ void __launch_bounds__(WS_THREADS, 1)
gr_matmul_q_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ MqArgs args, int64_t rows,
                   u64 mask) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself (keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sStage = smem;
  constexpr int MQ_STAGES = MqLayout<QM>::ST;
  uint8_t* sB = smem + MqLayout<QM>::OFF_B;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + MqLayout<QM>::OFF_BAR);
  uint64_t* raw_full = bars;
  uint64_t* limb_full = bars + MQ_STAGES;
  uint64_t* empty = bars + 2 * MQ_STAGES;
  uint64_t* tfull = bars + 3 * MQ_STAGES;      // [2] per TMEM buffer
  uint64_t* tempty = tfull + 2;                // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Q = args.q;

  const int kmax = args.k16 ? 16 : TC_D;
  for (int q = 0; q < Q; ++q) {
    const u64* M = args.M[q];
    uint8_t* dst = sB + q * BALL_BYTES;
    for (int e = tid; e < TC_D * TC_D; e += WS_THREADS) {
      const int k = e / TC_D, n = e % TC_D;
      const int h = n / DB_HALF, c = n % DB_HALF;
      const u64 v = k < kmax ? M[e] : 0ull;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        dst[core_off(256 * h + DB_HALF * j + c, k, BALL_ROWS / 8)] = uint8_t(v >> (8 * j));
    }
  }
  if (tid == 0) {
    for (int i = 0; i < MQ_STAGES; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&limb_full[i], W_CONV * 32);
      mbar_init(&empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], W_EPI * 32);
    }
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
  const int64_t my_tiles = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int upt = args.k16 ? 1 : 2;                  // K-units per tile
  const int64_t nunits = my_tiles * upt;
  const int pieces = 2 * Q;

  if (warp == W_EPI + W_CONV) {
    // ------------------------------ TMA producer
    if (lane == 0) {
      for (int64_t g = 0; g < nunits; ++g) {
        const int st = int(g % MQ_STAGES);
        if (g >= MQ_STAGES) mbar_wait(&empty[st], uint32_t((g / MQ_STAGES - 1) & 1));
        const int64_t t = blockIdx.x + (g / upt) * gridDim.x;
        const int kh = int(g % upt);
        uint8_t* dst = sStage + st * RAW_BYTES;
        mbar_expect_tx(&raw_full[st], upt == 2 ? RAW_BYTES : RAW_BYTES / 2);
        tma_load_2d(dst, &tm, kh * TC_KH, int(t * TC_ROWS), &raw_full[st]);
        if (upt == 2) tma_load_2d(dst + RAW_BYTES / 2, &tm, kh * TC_KH + 16, int(t * TC_ROWS), &raw_full[st]);
      }
    }
    __syncwarp();
  } else if (warp >= W_EPI && warp < W_EPI + W_CONV) {
    // ------------------------------ converters (in place)
    const int ct = tid - W_EPI * 32;
    const int r = ct & (TC_ROWS - 1), c = ct >> 7;
    const int sw = r & 7;
    for (int64_t g = 0; g < nunits; ++g) {
      const int st = int(g % MQ_STAGES);
      mbar_wait(&raw_full[st], uint32_t((g / MQ_STAGES) & 1));
      uint8_t* stage = sStage + st * RAW_BYTES;
      const uint8_t* src = stage + c * (RAW_BYTES / 2) + r * 128;
      uint32_t x[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + ((q ^ sw) << 4));
        x[4 * q + 0] = v.x;
        x[4 * q + 1] = v.y;
        x[4 * q + 2] = v.z;
        x[4 * q + 3] = v.w;
      }
      conv_named_sync();
      uint8_t* dst = stage + core_off(r, c * 16, TC_ROWS / 8);
      uint4 pk[8];
      split_limbs16(x, pk);
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(dst + i * LIMB_PLANE) = pk[i];
      fence_async_smem();
      mbar_arrive(&limb_full[st]);
    }
  } else if (warp == W_EPI + W_CONV + 1) {
    // ------------------------------ MMA issuer: pieces p = (q, h), buffer p & 1
    uint32_t tph[2] = {0, 0};
    int64_t use = 0;                                  // pieces issued so far (buffer uses)
    for (int64_t g0 = 0; g0 < nunits; g0 += upt) {
      for (int p = 0; p < pieces; ++p, ++use) {
        const int b = int(use & 1);
        if (use >= 2) {
          mbar_wait(&tempty[b], tph[b]);
          tph[b] ^= 1;
        }
        const int q = p >> 1, h = p & 1;
        for (int kh = 0; kh < upt; ++kh) {
          const int64_t g = g0 + kh;
          const int st = int(g % MQ_STAGES);
          if (p == 0) mbar_wait(&limb_full[st], uint32_t((g / MQ_STAGES) & 1));
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a0 = smem_u32(sStage + st * RAW_BYTES);
            const uint32_t b0 = smem_u32(sB + q * BALL_BYTES) + uint32_t((2 * kh * (BALL_ROWS / 8) + 32 * h) * 128);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint64_t ad = umma_desc(a0 + i * LIMB_PLANE, (TC_ROWS / 8) * 128, 128);
              const uint64_t bd = umma_desc(b0, (BALL_ROWS / 8) * 128, 128);
              mma_u8(tmem + uint32_t(256 * b + DB_HALF * i), ad, bd, idesc_u8(TC_ROWS, DB_HALF * (8 - i)),
                     (kh == 0 && i == 0) ? 0u : 1u);
            }
            if (p == pieces - 1) mma_commit(&empty[st]);
            if (kh == upt - 1) mma_commit(&tfull[b]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp < W_EPI) {
    // ------------------------------ epilogue
    uint32_t ph[2] = {0, 0};
    int64_t use = 0;
    const int quad = warp & 3, grp = warp >> 2;
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int p = 0; p < pieces; ++p, ++use) {
        const int b = int(use & 1), q = p >> 1, h = p & 1;
        mbar_wait(&tfull[b], ph[b]);
        ph[b] ^= 1;
        tc_fence_after();
        epi_half(tmem + (uint32_t(quad * 32) << 16) + uint32_t(256 * b), grp * (DB_HALF / 8), mask, args.out[q],
                 t * TC_ROWS + quad * 32, rows, DB_HALF * h, rq, cq);
        tc_fence_before();
        mbar_arrive(&tempty[b]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// d = 16: out = P0 . M0 (+ P1 . M1) with K = 16 per operand, so the two
// operands K-concatenate into ONE kind::i8 K-step of 32: a unit is a tile of
// 128 rows, raw = two TMA boxes (P0's and P1's 16 coefficients of the rows),
// B = [M0; M1] limb planes N-concatenated (row n' = 16 j + n, K = 32 bytes).
// 8 MMAs of N = 16 (8 - i) per tile into 8 x 16 = 128 TMEM columns; four such
// accumulators rotate so the MMAs of later tiles overlap the epilogue.
// ---------------------------------------------------------------------------
constexpr int T16_D = 16;
constexpr int T16_RAW = TC_ROWS * 2 * T16_D * 8;          // 32 KB (two 16 KB boxes)
constexpr int T16_LIMB_PLANE = TC_ROWS * 2 * T16_D;       // 4 KB (128 rows x 32 B)
constexpr int T16_LIMB = 8 * T16_LIMB_PLANE;              // 32 KB
constexpr int T16_BROWS = 8 * T16_D;                      // 128
constexpr int T16_B = T16_BROWS * 2 * T16_D;              // 4 KB
constexpr int T16_RAW_STAGES = 3, T16_LIMB_STAGES = 2;
constexpr int T16_OFF_LIMB = T16_RAW_STAGES * T16_RAW;
constexpr int T16_OFF_B = T16_OFF_LIMB + T16_LIMB_STAGES * T16_LIMB;
constexpr int T16_OFF_BAR = T16_OFF_B + T16_B;
constexpr int T16_SMEM = T16_OFF_BAR + 256 + 1024;
constexpr int T16_EPI = 4, T16_CONV = 8;
constexpr int T16_ACC = 4, T16_ACC_COLS = 128;            // TMEM accumulator buffers (8 x 16 columns each)
constexpr int T16_THREADS = (T16_EPI + T16_CONV + 2) * 32;

__global__ void __launch_bounds__(T16_THREADS, 1)
gr_matmul2_tc16_kernel(const __grid_constant__ Mm2Jobs J, const u64* __restrict__ M0, const u64* __restrict__ M1,
                       u64 mask) {
  const int nops = J.nops;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself (keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sRaw = smem;
  uint8_t* sLimb = smem + T16_OFF_LIMB;
  uint8_t* sB = smem + T16_OFF_B;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T16_OFF_BAR);
  uint64_t* raw_full = bars;         // [3]
  uint64_t* raw_empty = bars + 3;    // [3]
  uint64_t* limb_full = bars + 6;    // [2]
  uint64_t* limb_empty = bars + 8;   // [2]
  uint64_t* tfull = bars + 10;       // [4] one per TMEM accumulator buffer
  uint64_t* tempty = bars + 14;      // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // B: row n' = 16 j + n, k < 16 from M0, k >= 16 from M1 (zero if absent)
  for (int e = tid; e < 2 * T16_D * T16_D; e += T16_THREADS) {
    const int k = e / T16_D, n = e % T16_D;
    const u64 v = k < T16_D ? M0[k * T16_D + n] : (nops > 1 ? M1[(k - T16_D) * T16_D + n] : 0ull);
#pragma unroll
    for (int j = 0; j < 8; ++j) sB[core_off(j * T16_D + n, k, T16_BROWS / 8)] = uint8_t(v >> (8 * j));
  }
  if (tid == 0) {
    for (int i = 0; i < T16_RAW_STAGES; ++i) {
      mbar_init(&raw_full[i], 1);
      mbar_init(&raw_empty[i], T16_CONV * 32);
    }
    for (int i = 0; i < T16_LIMB_STAGES; ++i) {
      mbar_init(&limb_full[i], T16_CONV * 32);
      mbar_init(&limb_empty[i], 1);
    }
    for (int b = 0; b < T16_ACC; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], T16_EPI * 32);
    }
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
  const int64_t ntiles = J.tile0[J.njobs];
  const int64_t nunits = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;

  if (warp == T16_EPI + T16_CONV) {
    // ------------------------------ TMA producer
    if (lane == 0) {
      for (int64_t u = 0; u < nunits; ++u) {
        const int st = int(u % T16_RAW_STAGES);
        if (u >= T16_RAW_STAGES) mbar_wait(&raw_empty[st], uint32_t((u / T16_RAW_STAGES - 1) & 1));
        const int64_t t = blockIdx.x + u * gridDim.x;
        const int j = mm2_job(J, t);
        const int y = int((t - J.tile0[j]) * TC_ROWS);
        uint8_t* dst = sRaw + st * T16_RAW;
        mbar_expect_tx(&raw_full[st], uint32_t(nops * (T16_RAW / 2)));
        tma_load_2d(dst, &J.tm[j][0], 0, y, &raw_full[st]);
        if (nops > 1) tma_load_2d(dst + T16_RAW / 2, &J.tm[j][1], 0, y, &raw_full[st]);
      }
    }
    __syncwarp();
  } else if (warp >= T16_EPI && warp < T16_EPI + T16_CONV) {
    // ------------------------------ converters: thread = (row r, operand box c)
    const int ct = tid - T16_EPI * 32;
    const int r = ct & (TC_ROWS - 1), c = ct >> 7;
    const int sw = r & 7;
    for (int64_t u = 0; u < nunits; ++u) {
      const int st = int(u % T16_RAW_STAGES), ls = int(u % T16_LIMB_STAGES);
      mbar_wait(&raw_full[st], uint32_t((u / T16_RAW_STAGES) & 1));
      uint32_t x[32];
      if (c < nops) {
        const uint8_t* src = sRaw + st * T16_RAW + c * (T16_RAW / 2) + r * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 v = *reinterpret_cast<const uint4*>(src + ((q ^ sw) << 4));
          x[4 * q + 0] = v.x;
          x[4 * q + 1] = v.y;
          x[4 * q + 2] = v.z;
          x[4 * q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q) x[q] = 0;
      }
      fence_async_smem();   // generic-proxy reads before the next TMA write (WAR)
      mbar_arrive(&raw_empty[st]);
      if (u >= T16_LIMB_STAGES) mbar_wait(&limb_empty[ls], uint32_t((u / T16_LIMB_STAGES - 1) & 1));
      uint8_t* dst = sLimb + ls * T16_LIMB + core_off(r, c * 16, TC_ROWS / 8);
      uint4 pk[8];
      split_limbs16(x, pk);
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(dst + i * T16_LIMB_PLANE) = pk[i];
      fence_async_smem();
      mbar_arrive(&limb_full[ls]);
    }
  } else if (warp == T16_EPI + T16_CONV + 1) {
    // ------------------------------ MMA issuer
    for (int64_t u = 0; u < nunits; ++u) {
      const int ls = int(u % T16_LIMB_STAGES), b = int(u % T16_ACC);
      if (u >= T16_ACC) mbar_wait(&tempty[b], uint32_t((u / T16_ACC - 1) & 1));
      mbar_wait(&limb_full[ls], uint32_t((u / T16_LIMB_STAGES) & 1));
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sLimb + ls * T16_LIMB);
        const uint32_t b0 = smem_u32(sB);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint64_t ad = umma_desc(a0 + i * T16_LIMB_PLANE, (TC_ROWS / 8) * 128, 128);
          const uint64_t bd = umma_desc(b0, (T16_BROWS / 8) * 128, 128);
          mma_u8(tmem + uint32_t(T16_ACC_COLS * b + T16_D * i), ad, bd, idesc_u8(TC_ROWS, T16_D * (8 - i)),
                 i ? 1u : 0u);
        }
        mma_commit(&limb_empty[ls]);
        mma_commit(&tfull[b]);
      }
      __syncwarp();
    }
  } else if (warp < T16_EPI) {
    // ------------------------------ epilogue: warp e = TMEM lane quadrant e
    // (16-lane x 8-column loads: 4 threads per row, 64-byte row segments)
    const int rq = lane >> 2, cq = 2 * (lane & 3);
    for (int64_t u = 0; u < nunits; ++u) {
      const int b = int(u % T16_ACC);
      const int64_t t = blockIdx.x + u * gridDim.x;
      const int j = mm2_job(J, t);
      const int64_t lt = t - J.tile0[j];
      const int64_t rows = J.rows[j];
      u64* __restrict__ out = J.out[j];
      mbar_wait(&tfull[b], uint32_t((u / T16_ACC) & 1));
      tc_fence_after();
#pragma unroll 1
      for (int it = 0; it < 2 * (T16_D / 8); ++it) {
        const int lg = it & 1, c0 = 8 * (it >> 1);
        const uint32_t taddr = tmem + (uint32_t(warp * 32 + lg * 16) << 16) + uint32_t(T16_ACC_COLS * b + c0);
        uint32_t v[8][4];
#pragma unroll
        for (int s = 0; s < 8; ++s) tmem_ld_16x256(taddr + uint32_t(T16_D * s), v[s]);
        tmem_wait_ld();
        u64 acc[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          acc[q] = recombine8(v[0][q], v[1][q], v[2][q], v[3][q], v[4][q], v[5][q], v[6][q], v[7][q]) & mask;
        const int64_t row = lt * TC_ROWS + warp * 32 + lg * 16 + rq;
        if (row < rows)
          *reinterpret_cast<ulonglong2*>(out + row * T16_D + c0 + cq) = make_ulonglong2(acc[0], acc[1]);
        if (row + 8 < rows)
          *reinterpret_cast<ulonglong2*>(out + (row + 8) * T16_D + c0 + cq) = make_ulonglong2(acc[2], acc[3]);
      }
      tc_fence_before();
      mbar_arrive(&tempty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// host: tensor maps (driver entry point fetched through the runtime, so the
// library needs no -lcuda)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool make_rows_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t rs_words, int box_rows, int width) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return false;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  cuuint64_t dims[2] = {cuuint64_t(width), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(rs_words * 8)};
  cuuint32_t box[2] = {16u, cuuint32_t(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace r3

using namespace r3;

static int mm2_launch(const Mm2Jobs& J, const u64* M0, const u64* M1, uint64_t mask, cudaStream_t s) {
  const int64_t tiles = J.tile0[J.njobs];
  const unsigned grid = unsigned(tiles < num_sms() ? tiles : num_sms());
  ensure_smem(gr_matmul2_db_kernel, DB_SMEM);
  gr_matmul2_db_kernel<<<grid, WS_THREADS, DB_SMEM, s>>>(J, M0, M1, mask);
  return check_launch("r3_gr_matmul2_tc");
}

extern "C" int r3_gr_matmul2_tc(const uint64_t* p0, int64_t rs0, int64_t nv0, const uint64_t* p1, int64_t rs1,
                                int64_t nv1, const uint64_t* M0, const uint64_t* M1, uint64_t* out, int64_t rows,
                                uint64_t mask, void* stream) {
  if (!p0 || !M0 || rows < 0 || ((rs0 | rs1) & 1) || ((uintptr_t(p0) | uintptr_t(p1)) & 15) ||
      (p1 && !M1)) {
    set_error("r3_gr_matmul2_tc: bad arguments (need 16-byte aligned rows)");
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  if (rows > (int64_t(1) << 31) - TC_ROWS) {
    set_error("r3_gr_matmul2_tc: rows %lld exceed the TMA coordinate range", (long long)rows);
    return R3_ERR_ARG;
  }
  // operands with no valid rows contribute zero: drop them
  const uint64_t* P[2] = {p0, p1};
  const uint64_t* Ms[2] = {M0, M1};
  int64_t rs[2] = {rs0, rs1}, nv[2] = {nv0 < rows ? nv0 : rows, nv1 < rows ? nv1 : rows};
  int nops = 0;
  const uint64_t* Pk[2];
  const uint64_t* Mk[2];
  int64_t rsk[2], nvk[2];
  for (int q = 0; q < 2; ++q) {
    if (P[q] && nv[q] > 0) {
      Pk[nops] = P[q];
      Mk[nops] = Ms[q];
      rsk[nops] = rs[q] > 0 ? rs[q] : TC_D;
      nvk[nops] = nv[q];
      ++nops;
    }
  }
  if (nops == 0) {
    cudaMemsetAsync(out, 0, size_t(rows) * TC_D * 8, as_stream(stream));
    return check_launch("r3_gr_matmul2_tc(zero)");
  }
  Mm2Jobs J;
  J.njobs = 1;
  J.nops = nops;
  for (int q = 0; q < nops; ++q) {
    if (!make_rows_tmap(&J.tm[0][q], Pk[q], nvk[q], rsk[q], TC_ROWS)) {
      set_error("r3_gr_matmul2_tc: cuTensorMapEncodeTiled failed");
      return R3_ERR_CUDA;
    }
  }
  if (nops == 1) J.tm[0][1] = J.tm[0][0];
  J.out[0] = (u64*)out;
  J.rows[0] = rows;
  J.tile0[0] = 0;
  J.tile0[1] = (rows + TC_ROWS - 1) / TC_ROWS;
  return mm2_launch(J, (const u64*)Mk[0], (const u64*)(nops > 1 ? Mk[1] : Mk[0]), mask, as_stream(stream));
}

// Jobs of a multi launch (both operands present, >= 1 valid row each).
static int mm2_jobs(Mm2Jobs& J, const char* what, int d, int njobs, const uint64_t* const* p0, const int64_t* rs0,
                    const int64_t* nv0, const uint64_t* const* p1, const int64_t* rs1, const int64_t* nv1,
                    const uint64_t* M0, const uint64_t* M1, uint64_t* const* outs, const int64_t* rows) {
  if (njobs < 1 || njobs > MM2_MAX_JOBS || !p0 || !p1 || !rs0 || !rs1 || !nv0 || !nv1 || !M0 || !M1 || !outs ||
      !rows) {
    set_error("%s: bad arguments (1..%d jobs)", what, MM2_MAX_JOBS);
    return R3_ERR_ARG;
  }
  J.njobs = njobs;
  J.nops = 2;
  J.tile0[0] = 0;
  for (int j = 0; j < njobs; ++j) {
    const int64_t r = rows[j];
    const int64_t n0 = nv0[j] < r ? nv0[j] : r, n1 = nv1[j] < r ? nv1[j] : r;
    if (r < 1 || r > (int64_t(1) << 31) - TC_ROWS || !p0[j] || !p1[j] || !outs[j] || n0 < 1 || n1 < 1 ||
        ((rs0[j] | rs1[j]) & 1) || ((uintptr_t(p0[j]) | uintptr_t(p1[j])) & 15)) {
      set_error("%s: job %d: bad operand (rows %lld, valid %lld/%lld, 16-byte aligned rows)", what, j, (long long)r,
                (long long)n0, (long long)n1);
      return R3_ERR_ARG;
    }
    if (!make_rows_tmap(&J.tm[j][0], p0[j], n0, rs0[j] > 0 ? rs0[j] : d, TC_ROWS, d) ||
        !make_rows_tmap(&J.tm[j][1], p1[j], n1, rs1[j] > 0 ? rs1[j] : d, TC_ROWS, d)) {
      set_error("%s: cuTensorMapEncodeTiled failed", what);
      return R3_ERR_CUDA;
    }
    J.out[j] = (u64*)outs[j];
    J.rows[j] = r;
    J.tile0[j + 1] = J.tile0[j] + (r + TC_ROWS - 1) / TC_ROWS;
  }
  return R3_OK;
}

static int mm16_launch(const Mm2Jobs& J, const u64* M0, const u64* M1, uint64_t mask, cudaStream_t s) {
  const int64_t tiles = J.tile0[J.njobs];
  const unsigned grid = unsigned(tiles < num_sms() ? tiles : num_sms());
  ensure_smem(gr_matmul2_tc16_kernel, T16_SMEM);
  gr_matmul2_tc16_kernel<<<grid, T16_THREADS, T16_SMEM, s>>>(J, M0, M1, mask);
  return check_launch("r3_gr_matmul2_tc16");
}

extern "C" int r3_gr_matmul2_tc_multi(int njobs, const uint64_t* const* p0, const int64_t* rs0,
                                      const int64_t* nv0, const uint64_t* const* p1, const int64_t* rs1,
                                      const int64_t* nv1, const uint64_t* M0, const uint64_t* M1,
                                      uint64_t* const* outs, const int64_t* rows, uint64_t mask, void* stream) {
  Mm2Jobs J;
  const int rc = mm2_jobs(J, "r3_gr_matmul2_tc_multi", TC_D, njobs, p0, rs0, nv0, p1, rs1, nv1, M0, M1, outs, rows);
  return rc != R3_OK ? rc : mm2_launch(J, (const u64*)M0, (const u64*)M1, mask, as_stream(stream));
}

extern "C" int r3_gr_matmul2_tc16(const uint64_t* p0, int64_t rs0, int64_t nv0, const uint64_t* p1, int64_t rs1,
                                  int64_t nv1, const uint64_t* M0, const uint64_t* M1, uint64_t* out,
                                  int64_t rows, uint64_t mask, void* stream) {
  if (!p0 || !M0 || rows < 0 || ((rs0 | rs1) & 1) || ((uintptr_t(p0) | uintptr_t(p1)) & 15) || (p1 && !M1)) {
    set_error("r3_gr_matmul2_tc16: bad arguments (need 16-byte aligned rows)");
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  if (rows > (int64_t(1) << 31) - TC_ROWS) {
    set_error("r3_gr_matmul2_tc16: rows %lld exceed the TMA coordinate range", (long long)rows);
    return R3_ERR_ARG;
  }
  const uint64_t* P[2] = {p0, p1};
  const uint64_t* Ms[2] = {M0, M1};
  int64_t rs[2] = {rs0, rs1}, nv[2] = {nv0 < rows ? nv0 : rows, nv1 < rows ? nv1 : rows};
  int nops = 0;
  const uint64_t* Pk[2];
  const uint64_t* Mk[2];
  int64_t rsk[2], nvk[2];
  for (int q = 0; q < 2; ++q) {
    if (P[q] && nv[q] > 0) {
      Pk[nops] = P[q];
      Mk[nops] = Ms[q];
      rsk[nops] = rs[q] > 0 ? rs[q] : T16_D;
      nvk[nops] = nv[q];
      ++nops;
    }
  }
  if (nops == 0) {
    cudaMemsetAsync(out, 0, size_t(rows) * T16_D * 8, as_stream(stream));
    return check_launch("r3_gr_matmul2_tc16(zero)");
  }
  Mm2Jobs J;
  J.njobs = 1;
  J.nops = nops;
  for (int q = 0; q < nops; ++q) {
    if (!make_rows_tmap(&J.tm[0][q], Pk[q], nvk[q], rsk[q], TC_ROWS, T16_D)) {
      set_error("r3_gr_matmul2_tc16: cuTensorMapEncodeTiled failed");
      return R3_ERR_CUDA;
    }
  }
  if (nops == 1) J.tm[0][1] = J.tm[0][0];
  J.out[0] = (u64*)out;
  J.rows[0] = rows;
  J.tile0[0] = 0;
  J.tile0[1] = (rows + TC_ROWS - 1) / TC_ROWS;
  return mm16_launch(J, (const u64*)Mk[0], (const u64*)(nops > 1 ? Mk[1] : Mk[0]), mask, as_stream(stream));
}

extern "C" int r3_gr_matmul2_tc16_multi(int njobs, const uint64_t* const* p0, const int64_t* rs0,
                                        const int64_t* nv0, const uint64_t* const* p1, const int64_t* rs1,
                                        const int64_t* nv1, const uint64_t* M0, const uint64_t* M1,
                                        uint64_t* const* outs, const int64_t* rows, uint64_t mask, void* stream) {
  Mm2Jobs J;
  const int rc = mm2_jobs(J, "r3_gr_matmul2_tc16_multi", T16_D, njobs, p0, rs0, nv0, p1, rs1, nv1, M0, M1, outs,
                          rows);
  return rc != R3_OK ? rc : mm16_launch(J, (const u64*)M0, (const u64*)M1, mask, as_stream(stream));
}

static int mq_launch(const MqArgs& a, const void* p, int64_t rs, int width, int64_t rows, u64 mask, void* stream,
                     const char* who) {
  CUtensorMap tm;
  if (!make_rows_tmap(&tm, p, rows, rs, TC_ROWS, width)) {
    set_error("%s: cuTensorMapEncodeTiled failed", who);
    return R3_ERR_CUDA;
  }
  const int64_t tiles = (rows + TC_ROWS - 1) / TC_ROWS;
  const unsigned grid = unsigned(tiles < num_sms() ? tiles : num_sms());
  if (a.q <= 2) {
    ensure_smem(gr_matmul_q_kernel<2>, MqLayout<2>::SMEM);
    gr_matmul_q_kernel<2><<<grid, WS_THREADS, MqLayout<2>::SMEM, as_stream(stream)>>>(tm, a, rows, mask);
  } else {
    ensure_smem(gr_matmul_q_kernel<4>, MqLayout<4>::SMEM);
    gr_matmul_q_kernel<4><<<grid, WS_THREADS, MqLayout<4>::SMEM, as_stream(stream)>>>(tm, a, rows, mask);
  }
  return check_launch(who);
}

extern "C" int r3_gr_matmul_q_tc(const uint64_t* p, int64_t rs, int64_t rows, const uint64_t* const* Ms,
                                 uint64_t* const* outs, int q, uint64_t mask, void* stream) {
  if (!p || !Ms || !outs || q < 1 || q > MQ_MAX || rows < 0 || (rs & 1) || (uintptr_t(p) & 15)) {
    set_error("r3_gr_matmul_q_tc: bad arguments (1 <= q <= 4, 16-byte aligned rows)");
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  if (rows > (int64_t(1) << 31) - TC_ROWS) {
    set_error("r3_gr_matmul_q_tc: rows %lld exceed the TMA coordinate range", (long long)rows);
    return R3_ERR_ARG;
  }
  MqArgs a{};
  a.q = q;
  for (int i = 0; i < q; ++i) {
    if (!Ms[i] || !outs[i]) {
      set_error("r3_gr_matmul_q_tc: null matrix or output");
      return R3_ERR_ARG;
    }
    a.M[i] = reinterpret_cast<const u64*>(Ms[i]);
    a.out[i] = reinterpret_cast<u64*>(outs[i]);
  }
  return mq_launch(a, p, rs > 0 ? rs : TC_D, TC_D, rows, mask, stream, "r3_gr_matmul_q_tc");
}

// out[j] = sum_{a < 16} p[16 j + a] K[a] for a 16 x 64 matrix K: the
// level-4 rows of the y side of a multiplication log with blocks of 16,
// kappa_a times base elements (r3_vfy_line_b_const's arithmetic as a K = 16
// byte-limb GEMM, so the step is bound by the row bytes, not by the CUDA
// cores' 1024 multiply-adds per row and component).  p: rows x 16 words.
extern "C" int r3_gr_matmul_k16_tc(const uint64_t* p, int64_t rows, const uint64_t* K, uint64_t* out,
                                   uint64_t mask, void* stream) {
  if (!p || !K || !out || rows < 0 || (uintptr_t(p) & 15)) {
    set_error("r3_gr_matmul_k16_tc: bad arguments (16-byte aligned rows)");
    return R3_ERR_ARG;
  }
  if (rows == 0) return R3_OK;
  if (rows > (int64_t(1) << 31) - TC_ROWS) {
    set_error("r3_gr_matmul_k16_tc: rows %lld exceed the TMA coordinate range", (long long)rows);
    return R3_ERR_ARG;
  }
  MqArgs a{};
  a.q = 1;
  a.k16 = 1;
  a.M[0] = reinterpret_cast<const u64*>(K);
  a.out[0] = reinterpret_cast<u64*>(out);
  return mq_launch(a, p, 16, 16, rows, mask, stream, "r3_gr_matmul_k16_tc");
}
