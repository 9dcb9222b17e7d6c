// Base fold of a multiplication log on the tensor cores (d = 64), all
// simulated parties in one pass over the r^(4j) table.
//
// The first two reductions of Pi_mulv come straight from the base log
// (vfy2.cu): per party and block j of four elements the 16 scalar leg
// products s^{ab}_j = sum_t c_t x_t[4j+a] y_t[4j+b] and the z values
// z_c[4j+a] are weighted by the public row r^(4j):
//     acc'[p][a*4+b] = sum_j s^{ab}_j r^(4j),   zraw[p][c*4+a] = sum_j z_c[4j+a] r^(4j).
// That is ONE matrix product A^T B over the blocks j, with A's 128 columns
// the features (party p: 32 p + q, q < 16 the s products, 16 + c*4 + a the
// z values) and B the table rows (N = 64 coefficients), computed as the 36
// byte-limb products of kind::i8 MMAs (12 per K-step, N-concatenated), as in
// the level fold (lf_tc.cu).  The converter warps compute the s products
// from the base shares and split them into limb planes; B arrives by TMA.
// A CTA's K range is <= 16384 blocks (exact low diagonals, tc.cu).  The
// epilogue recombines each feature row and adds it to its party's output.
#include "tc_common.cuh"

namespace r3 {

constexpr int BF_BK = 32;                       // blocks j per K-step
constexpr int BF_A_PLANE = 128 * BF_BK;         // 4 KB
constexpr int BF_B_PLANE = 64 * BF_BK;          // 2 KB
constexpr int BF_A_TILE = 8 * BF_A_PLANE;       // 32 KB
constexpr int BF_B_TILE = 8 * BF_B_PLANE;       // 16 KB
constexpr int BF_BOX = 16 * 8 * BF_BK;          // TMA box: 16 u64 x 32 rows = 4 KB
constexpr int BF_RAW = 4 * BF_BOX;              // one K-step of table rows: 16 KB
constexpr int BF_STAGES = 3;
constexpr int BF_CONV = 12 * 32;                // 256 A tasks + 128 B tasks per K-step
constexpr int BF_THREADS = 4 * 32 + BF_CONV + 2 * 32;
constexpr int64_t BF_MAX_K = 16384;
constexpr int BF_MAX_SLOTS = 6;                 // distinct x / y / z arrays of a party

// Shared-memory layout.  B = 4: three raw stages of table rows.  B = 8, 16
// ("wide"): two raw stages, each the table rows plus the base-log arrays the
// work item reads in the K-step, all by TMA (so the converters never wait on
// global loads): B = 8 all of the party's arrays (x / y / z, <= 6 x 2 KB),
// B = 16 either a party's x / y arrays (<= 4 x 4 KB) or, for the one z
// item of a chunk, every party's distinct z arrays (<= 6 x 4 KB).  A log
// array is viewed as rows of 16 words (128 B) with the 128-byte swizzle,
// which makes the converters' per-block reads bank-conflict free.
// Work items per K chunk: B = 8 one per party (64 + 8 nz features fill the
// 128 MMA rows); B = 16 two per party (256 s products: rows a < 8 and
// a >= 8) plus ONE z item for all parties (16 features per distinct z
// array).
// D = extension degree (table row width): 64 or 16.  The table rows of a
// K-step are D / 16 TMA boxes; the B operand is D columns per limb plane.
template <int B, int D = 64>
struct BfLayout {
  static constexpr bool WIDE = B >= 8;
  // raw (TMA) stages vs limb stages: the converters, not the MMA, wait
  // (ncu r04o: 13 % of the q16 kernel's stall samples on raw_full, 2 % on
  // the limb barriers), so the wide D = 64 layouts trade a limb stage for
  // a third raw stage; D = 16 has room for four raw stages and three limb
  // stages
  static constexpr int RS = !WIDE ? 3 : (D == 16 ? 4 : 3);
  static constexpr int STAGES = (WIDE && D == 64) ? 2 : BF_STAGES;
  static constexpr int NBOX = D / 16;
  static constexpr int RAW = NBOX * BF_BOX;     // one K-step of table rows
  static constexpr int B_PLANE = D * BF_BK;
  static constexpr int B_TILE = 8 * B_PLANE;
  static constexpr int SLOT = BF_BK * B * 8;    // one array over a K-step (TMA box, 128B swizzle)
  static constexpr int NSLOT = 6;               // B = 16: <= 4 x / y arrays, or the z item's <= 6
  static constexpr int RAWST = (RAW + (WIDE ? NSLOT * SLOT : 0) + 1023) / 1024 * 1024;
  static constexpr int OFF_LIMB = RS * RAWST;
  static constexpr int OFF_BAR = OFF_LIMB + STAGES * (BF_A_TILE + B_TILE);
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
};
static_assert(BfLayout<16>::SMEM <= 232448, "base fold q16 shared memory");
static_assert(BfLayout<8>::SMEM <= 232448, "base fold q8 shared memory");
static_assert(BfLayout<4>::SMEM <= 232448, "base fold q4 shared memory");
static_assert(BfLayout<16, 16>::SMEM <= 232448, "base fold q16 (d = 16) shared memory");
static_assert(BfLayout<8, 16>::SMEM <= 232448, "base fold q8 (d = 16) shared memory");

struct BfParty {
  const u64* x[3];
  const u64* y[3];
  const u64* z[2];
  u64 coef[3];
  int nterms, nz;
  int64_t zs;
  u64* acc;    // B^2 x 64
  u64* zraw;   // (B nz) x 64
  // wide B: the distinct x / y arrays (slot[0, nxy)) and z arrays
  // (slot[nxy, nxy + nz)), bulk-copied per K-step, and each term's slots
  const u64* slot[BF_MAX_SLOTS];
  int nxy;
  int sx[3], sy[3];
};

struct BfArgs {
  CUtensorMap pw4;
  CUtensorMap lmap[3][BF_MAX_SLOTS];   // wide B: the parties' base-log arrays as 16-word rows
  // B = 16: ONE z item per K chunk for every party -- the distinct z arrays
  // (the honest m is shared by P1 and P2), their maps and where each one's
  // sums go (party, component)
  CUtensorMap zmap[BF_MAX_SLOTS];
  const u64* zslot[BF_MAX_SLOTS];
  int nzs;
  int zdst_n[BF_MAX_SLOTS], zdst_p[BF_MAX_SLOTS][2], zdst_c[BF_MAX_SLOTS][2];
  int per;     // work items per K chunk
  BfParty p[3];
  int np;
  int vec;     // every base-log pointer 16-byte aligned: 128-bit loads
  int64_t N, nblk, kc;
};


// B = 4: the three parties' features share the 128 MMA rows (party p:
// 32 p + q).  B = 8: 64 s products + 8 nz z values per party, so a work item
// is (K chunk, party) and the np items of one chunk are adjacent in the
// grid (co-resident: the table rows come from HBM once, L2 for the others).
template <int B, int D>
__global__ void __launch_bounds__(BF_THREADS, 1)
base_fold_tc_kernel(const __grid_constant__ BfArgs args) {
  using L = BfLayout<B, D>;
  constexpr int RS = L::RS;
  constexpr int NST = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by offsetting the shared array itself (keeps the shared
  // address space visible to the compiler: LDS / STS instead of generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sRaw = smem;
  uint8_t* sA = smem + L::OFF_LIMB;
  uint8_t* sB = sA + NST * BF_A_TILE;   // B tiles: L::B_TILE each
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = bars + RS;
  uint64_t* full = bars + 2 * RS;
  uint64_t* empty = bars + 2 * RS + NST;
  uint64_t* tfull = bars + 2 * RS + 2 * NST;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // persistent: CTA b takes K-chunks (items) b, b + grid, ... of kc blocks;
  // unit g enumerates (item, K-step) in that order
  const int64_t nchunks = (args.nblk + args.kc - 1) / args.kc;
  const int per = B == 4 ? 1 : args.per;
  const int64_t nitems = nchunks * per;
  auto item_range = [&](int64_t it, int64_t& j0, int64_t& j1) {
    j0 = (it / per) * args.kc;
    j1 = min(args.nblk, j0 + args.kc);
  };
  // wide B: item -> (party, feature group).  B = 8: one item per party.
  // B = 16: items 2q, 2q + 1 of a chunk are party q's s rows a < 8 / a >= 8,
  // the last one the shared z item (party 0 stands in; group 2)
  auto item_party = [&](int64_t it) {
    const int r = int(it % per);
    return B == 4 ? 0 : (B == 8 ? r : (r < 2 * args.np ? r >> 1 : 0));
  };
  auto item_group = [&](int64_t it) {
    const int r = int(it % per);
    return B == 16 ? (r < 2 * args.np ? (r & 1) : 2) : 0;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], L::WIDE ? BF_CONV : 128);   // wide B: A threads read the log stage too
    }
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], BF_CONV);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
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
    // ---------------- TMA producer: table rows j of the K-step; wide B:
    // also the base-log rows of the arrays the item reads
    if (lane == 0) {
      int64_t g = 0;
      for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
        int64_t j0, j1;
        item_range(it, j0, j1);
        const int64_t nkb = (j1 - j0 + BF_BK - 1) / BF_BK;
        const int pi = item_party(it);
        const BfParty& P = args.p[pi];
        const int grp = item_group(it);
        // the arrays this item reads: B = 8 all of the party's, B = 16 its x /
        // y arrays (s groups) or every party's distinct z arrays (z item)
        const bool zitem = B == 16 && grp == 2;
        const int nsl = zitem ? args.nzs : (B == 16 ? P.nxy : P.nxy + P.nz);
        for (int64_t kb = 0; kb < nkb; ++kb, ++g) {
          const int rs = int(g % RS);
          if (g >= RS) mbar_wait(&raw_empty[rs], uint32_t((g / RS - 1) & 1));
          const int y = int(j0 + kb * BF_BK);
          // wide B: the K-step's 32 B elements of the arrays, unless the step
          // crosses the end of the log (the converters load those)
          const bool whole = L::WIDE && args.vec && (j0 + (kb + 1) * BF_BK) * B <= args.N;
          uint8_t* dst = sRaw + rs * L::RAWST;
          mbar_expect_tx(&raw_full[rs], uint32_t(L::RAW + (whole ? nsl * L::SLOT : 0)));
          for (int c = 0; c < L::NBOX; ++c)
            tma_load_2d(dst + c * BF_BOX, &args.pw4, c * 16, y, &raw_full[rs]);
          if (whole)
            for (int q = 0; q < nsl; ++q)
              tma_load_2d(dst + L::RAW + q * L::SLOT, zitem ? &args.zmap[q] : &args.lmap[pi][q], 0,
                          int(int64_t(y) * B / 16), &raw_full[rs]);
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 16) {
    // ---------------- converters: thread = (block k of the K-step, 16-feature chunk c)
    const int lt = threadIdx.x - 128;
    const bool isA = lt < 256;
    const int k = lt & 31;
    const int c = isA ? (lt >> 5) : ((lt - 256) >> 5);
    int64_t g = -1;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    // h: 0 = s products, 1 = z values, 2 = zero rows.  B = 8: chunk c < 4
    // holds s rows a = 2c, 2c + 1, chunk 4 the z values.  B = 16: s groups
    // hold row a = 8 grp + c per chunk, the z group z_c in chunk c < nz.
    const int grp = item_group(it);
    const int p = B == 4 ? c >> 1 : item_party(it);
    const int h = B == 4 ? (c & 1)
                  : B == 8 ? (c < 4 ? 0 : (c == 4 ? 1 : 2))
                           : (grp < 2 ? 0 : (c < args.nzs ? 1 : 2));
    const bool live = isA && p < args.np && h < 2;
    constexpr int NA = B == 8 ? 2 : 1;               // s rows per chunk (wide B)
    const int a0 = B == 8 ? 2 * c : 8 * grp + c;     // first s row of the chunk
    int64_t j0, j1;
    item_range(it, j0, j1);
    const int64_t nkb = (j1 - j0 + BF_BK - 1) / BF_BK;
    for (int64_t kb = 0; kb < nkb; ++kb) {
      ++g;
      const int st = int(g % NST);
      const int rs = int(g % RS);
      const int64_t j = j0 + kb * BF_BK + k;
      const bool ok = j < j1;
      u64 v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = 0;
      bool staged = false;
      if (L::WIDE && isA) {
        // the K-step's base-log arrays arrive with the table rows
        mbar_wait(&raw_full[rs], uint32_t((g / RS) & 1));
        staged = args.vec && (j0 + (kb + 1) * BF_BK) * B <= args.N;
        if (live && staged) {
          const BfParty& P = args.p[p];
          const uint8_t* lg = sRaw + rs * L::RAWST + L::RAW;
          // block k's 16-byte chunk ch of a slot: row k (B = 16) or k / 2
          // (B = 8, second half of the row for odd k), 128-byte swizzle
          const int rrow = B == 16 ? k : (k >> 1);
          const int cb = B == 16 ? 0 : (k & 1) * 4;
          auto chunk = [&](int slot, int ch) {
            return lg + slot * L::SLOT + rrow * 128 + (((cb + ch) ^ (rrow & 7)) << 4);
          };
          if (h == 0) {          // v[(a - a0) B + b] = sum_t c_t x_t[B j + a] y_t[B j + b]
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              if (t < P.nterms) {
                u64 cx[NA];
                if constexpr (NA == 2) {
                  const ulonglong2 xx = *reinterpret_cast<const ulonglong2*>(chunk(P.sx[t], a0 >> 1));
                  cx[0] = P.coef[t] * xx.x;
                  cx[NA - 1] = P.coef[t] * xx.y;
                } else {
                  cx[0] = P.coef[t] * *reinterpret_cast<const u64*>(chunk(P.sx[t], a0 >> 1) + (a0 & 1) * 8);
                }
#pragma unroll
                for (int q = 0; q < B / 2; ++q) {
                  const ulonglong2 yy = *reinterpret_cast<const ulonglong2*>(chunk(P.sy[t], q));
#pragma unroll
                  for (int a = 0; a < NA; ++a) {
                    v[a * B + 2 * q] += cx[a] * yy.x;
                    v[a * B + 2 * q + 1] += cx[a] * yy.y;
                  }
                }
              }
            }
          } else {               // z values: B = 8 v[cz 8 + a] (chunk 4), B = 16 v[a] (z slot c)
            const int zbase = B == 8 ? P.nxy : 0;   // B = 8: z arrays follow the party's x / y arrays
#pragma unroll
            for (int cz = 0; cz < (B == 8 ? 2 : 1); ++cz) {
              const int zc = B == 8 ? cz : c;
              if (zc < (B == 8 ? P.nz : args.nzs)) {
#pragma unroll
                for (int q = 0; q < B / 2; ++q) {
                  const ulonglong2 zz = *reinterpret_cast<const ulonglong2*>(chunk(zbase + zc, q));
                  v[cz * B + 2 * q] = zz.x, v[cz * B + 2 * q + 1] = zz.y;
                }
              }
            }
          }
        }
        fence_async_smem();   // generic-proxy reads before the next bulk write (WAR)
        mbar_arrive(&raw_empty[rs]);
      }
      if (isA) {
        if (live && ok && L::WIDE && !staged) {
          // the K-step crossing the end of the log: plain loads
          const BfParty& P = args.p[p];
          const int64_t i0 = int64_t(B) * j;
          if (h == 0) {
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              if (t < P.nterms) {
                u64 xv[NA], yv[B];
#pragma unroll
                for (int a = 0; a < NA; ++a) {
                  const int64_t i = i0 + a0 + a;
                  xv[a] = i < args.N ? __ldg(P.x[t] + i) : 0ull;
                }
#pragma unroll
                for (int b = 0; b < B; ++b) yv[b] = i0 + b < args.N ? __ldg(P.y[t] + i0 + b) : 0ull;
#pragma unroll
                for (int a = 0; a < NA; ++a) {
                  const u64 cx = P.coef[t] * xv[a];
#pragma unroll
                  for (int b = 0; b < B; ++b) v[a * B + b] += cx * yv[b];
                }
              }
            }
          } else {
#pragma unroll
            for (int cz = 0; cz < (B == 8 ? 2 : 1); ++cz) {
              const int zc = B == 8 ? cz : c;
              if (zc < (B == 8 ? P.nz : args.nzs)) {
                const u64* zp = B == 8 ? P.z[zc] : args.zslot[zc];
                const int64_t zst = B == 8 ? P.zs : 1;
#pragma unroll
                for (int a = 0; a < B; ++a)
                  v[cz * B + a] = i0 + a < args.N ? __ldg(zp + (i0 + a) * zst) : 0ull;
              }
            }
          }
        } else if (B == 4 && live && ok) {
          const BfParty& P = args.p[p];
          const int64_t i0 = 4 * j;
          if (h == 0) {
#pragma unroll
            for (int t = 0; t < 3; ++t) {
              if (t >= P.nterms) break;
              u64 xv[4], yv[4];
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                const bool in = i0 + a < args.N;
                xv[a] = in ? __ldg(P.x[t] + i0 + a) : 0ull;
                yv[a] = in ? __ldg(P.y[t] + i0 + a) : 0ull;
              }
#pragma unroll
              for (int a = 0; a < 4; ++a) {
                const u64 cx = P.coef[t] * xv[a];
#pragma unroll
                for (int b = 0; b < 4; ++b) v[a * 4 + b] += cx * yv[b];
              }
            }
          } else {
#pragma unroll
            for (int cz = 0; cz < 2; ++cz) {
              if (cz < P.nz) {
#pragma unroll
                for (int a = 0; a < 4; ++a)
                  v[cz * 4 + a] = i0 + a < args.N ? __ldg(P.z[cz] + (i0 + a) * P.zs) : 0ull;
              }
            }
          }
        }
      } else {
        mbar_wait(&raw_full[rs], uint32_t((g / RS) & 1));
        if (c < L::NBOX) {   // D = 16: one 16-coefficient chunk; the other B threads only keep the barriers
          const uint8_t* row = sRaw + rs * L::RAWST + c * BF_BOX + k * 128;
          const int sw = k & 7;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(row + ((q ^ sw) << 4));
            v[2 * q] = x.x;
            v[2 * q + 1] = x.y;
          }
        }
        fence_async_smem();   // generic-proxy reads before the next TMA write (WAR)
        mbar_arrive(&raw_empty[rs]);
      }
      uint4 pk[8];
      split_limbs16(v, pk);
      if (g >= NST) mbar_wait(&empty[st], uint32_t((g / NST - 1) & 1));
      // MN-major no-swizzle core layout: chunk stride 512 B, k-row stride 16 B
      uint8_t* dst = isA ? sA + st * BF_A_TILE : sB + st * L::B_TILE;
      const int plane = isA ? BF_A_PLANE : L::B_PLANE;
      const uint32_t off = uint32_t(c * 512 + k * 16);
      if (isA || c < L::NBOX) {
#pragma unroll
        for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(dst + i * plane + off) = pk[i];
      }
      fence_async_smem();
      mbar_arrive(&full[st]);
    }
    }
  } else if (warp == 4 + 12 + 1) {
    // ---------------- MMA issuer (as lf_tc: 12 N-concatenated limb MMAs per K-step)
    constexpr uint32_t IDESC_M128 = idesc_u8(128, 0) | (1u << 15) | (1u << 16);
    int64_t g = -1;
    uint32_t tph = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    int64_t j0, j1;
    item_range(it, j0, j1);
    const int64_t nkb = (j1 - j0 + BF_BK - 1) / BF_BK;
    if (it != blockIdx.x) {        // the epilogue has drained the previous item
      mbar_wait(tempty, tph);
      tph ^= 1;
    }
    for (int64_t kb = 0; kb < nkb; ++kb) {
      ++g;
      const int st = int(g % NST);
      mbar_wait(&full[st], uint32_t((g / NST) & 1));
      tc_fence_after();
      if (lane == 0) {
        const uint32_t a0 = smem_u32(sA + st * BF_A_TILE);
        const uint32_t b0 = smem_u32(sB + st * L::B_TILE);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint64_t ad = umma_desc(a0 + i * BF_A_PLANE, 128, 512);
#pragma unroll
          for (int n0 = 0; n0 < D * (8 - i); n0 += 256) {
            const int nn = D * (8 - i) - n0 < 256 ? D * (8 - i) - n0 : 256;
            const uint64_t bd = umma_desc(b0 + uint32_t(n0 / 16) * 512, 128, 512);
            mma_u8(tmem + uint32_t(i * D + n0), ad, bd, IDESC_M128 | (uint32_t(nn >> 3) << 17),
                   (kb == 0 && i == 0) ? 0u : 1u);
          }
        }
        mma_commit(&empty[st]);
      }
      __syncwarp();
    }
    if (lane == 0) mma_commit(tfull);
    __syncwarp();
    }
  } else if (warp < 4) {
    // ---------------- epilogue: TMEM lane f = feature (party f / 32, slot f % 32)
    uint32_t ph = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
      mbar_wait(tfull, ph);
      ph ^= 1;
      tc_fence_after();
      const int f = warp * 32 + lane;
      u64* dst = nullptr;
      u64* dst2 = nullptr;
      if (B == 4) {
        const int p = f >> 5, q = f & 31;
        const bool live = p < args.np && (q < 16 || q < 16 + 4 * args.p[p < 3 ? p : 0].nz);
        if (live) dst = q < 16 ? args.p[p].acc + q * D : args.p[p].zraw + (q - 16) * D;
      } else if (B == 8) {
        const BfParty& P = args.p[item_party(it)];
        if (f < 64) dst = P.acc + f * D;
        else if (f < 64 + 8 * P.nz) dst = P.zraw + (f - 64) * D;
      } else {
        const int grp = item_group(it);
        if (grp < 2) {
          dst = args.p[item_party(it)].acc + (128 * grp + f) * D;
        } else if ((f >> 4) < args.nzs) {
          // z slot f / 16 feeds one or two (party, component) sums
          const int zs = f >> 4, a = f & 15;
          dst = args.p[args.zdst_p[zs][0]].zraw + (16 * args.zdst_c[zs][0] + a) * D;
          if (args.zdst_n[zs] > 1) dst2 = args.p[args.zdst_p[zs][1]].zraw + (16 * args.zdst_c[zs][1] + a) * D;
        }
      }
      const bool live = dst != nullptr;
      const uint32_t lane_base = tmem + (uint32_t(warp * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 8) {
        uint32_t v[8][8];
#pragma unroll
        for (int s = 0; s < 8; ++s) tmem_ld8(lane_base + uint32_t(s * D + c0), v[s]);
        tmem_wait_ld();
        if (live) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            u64 P = 0;
#pragma unroll
            for (int s = 0; s < 8; ++s) P += u64(v[s][e]) << (8 * s);
            atomicAdd(reinterpret_cast<unsigned long long*>(dst + c0 + e), (unsigned long long)P);
            if (dst2) atomicAdd(reinterpret_cast<unsigned long long*>(dst2 + c0 + e), (unsigned long long)P);
          }
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

namespace {

template <int B, int D = 64>
int base_fold_tc_launch(int np, const int* nterms, const int64_t* coef, const uint64_t* const* xc,
                        const uint64_t* const* yc, const int* nz, const uint64_t* const* zc, const int64_t* zs,
                        int64_t N, const uint64_t* pw, uint64_t* const* acc, uint64_t* const* zraw,
                        cudaStream_t s, const char* what) {
  const int64_t nblk = (N + B - 1) / B;
  BfArgs args{};
  args.np = np;
  args.N = N;
  args.nblk = nblk;
  for (int q = 0; q < np; ++q) {
    BfParty& P = args.p[q];
    P.nterms = nterms[q];
    P.nz = nz[q];
    P.zs = zs[q];
    for (int t = 0; t < nterms[q]; ++t) {
      P.x[t] = reinterpret_cast<const u64*>(xc[3 * q + t]);
      P.y[t] = reinterpret_cast<const u64*>(yc[3 * q + t]);
      P.coef[t] = u64(coef[3 * q + t]);
    }
    for (int c = 0; c < nz[q]; ++c) P.z[c] = reinterpret_cast<const u64*>(zc[2 * q + c]);
    P.acc = reinterpret_cast<u64*>(acc[q]);
    P.zraw = reinterpret_cast<u64*>(zraw[q]);
  }
  uintptr_t align = 0;
  for (int q = 0; q < np; ++q) {
    for (int t = 0; t < args.p[q].nterms; ++t)
      align |= reinterpret_cast<uintptr_t>(args.p[q].x[t]) | reinterpret_cast<uintptr_t>(args.p[q].y[t]);
    for (int c = 0; c < args.p[q].nz; ++c) align |= reinterpret_cast<uintptr_t>(args.p[q].z[c]);
  }
  args.vec = (align & 15) == 0;
  if (BfLayout<B>::WIDE) {
    // distinct x / y arrays per party, then its z arrays (bulk-copied per K-step)
    for (int q = 0; q < np; ++q) {
      BfParty& P = args.p[q];
      auto slot_of = [&](const u64* a) {
        for (int s2 = 0; s2 < P.nxy; ++s2)
          if (P.slot[s2] == a) return s2;
        P.slot[P.nxy] = a;
        return P.nxy++;
      };
      for (int t = 0; t < P.nterms; ++t) P.sx[t] = slot_of(P.x[t]), P.sy[t] = slot_of(P.y[t]);
      if (P.nxy > 4) args.vec = 0;             // (<= 4 distinct x / y arrays in every leg form)
      for (int c = 0; c < P.nz; ++c) P.slot[P.nxy + c] = P.z[c];
      if (P.nz && P.zs != 1) args.vec = 0;
    }
    if (B == 16) {
      // the shared z item: distinct z arrays of all parties and their sums
      for (int q = 0; q < np; ++q) {
        const BfParty& P = args.p[q];
        for (int c = 0; c < P.nz; ++c) {
          int zs = 0;
          while (zs < args.nzs && args.zslot[zs] != P.z[c]) ++zs;
          if (zs == args.nzs) {
            if (args.nzs == BF_MAX_SLOTS || P.zs != 1) {
              set_error("%s: more than 6 distinct z arrays (or strided z)", what);
              return R3_ERR_ARG;
            }
            args.zslot[args.nzs] = P.z[c];
            args.zdst_n[args.nzs++] = 0;
          }
          if (args.zdst_n[zs] == 2) {
            set_error("%s: a z array shared by more than two parties", what);
            return R3_ERR_ARG;
          }
          args.zdst_p[zs][args.zdst_n[zs]] = q;
          args.zdst_c[zs][args.zdst_n[zs]++] = c;
        }
      }
      for (int zs = 0; zs < args.nzs && args.vec; ++zs)
        if (!make_rows_tmap(&args.zmap[zs], args.zslot[zs], N / 16, 16, BF_BK * B / 16, 16)) {
          set_error("%s: cuTensorMapEncodeTiled (z) failed", what);
          return R3_ERR_CUDA;
        }
    }
    // each array as floor(N / 16) rows of 16 words; a K-step's box: 32 blocks
    for (int q = 0; q < np && args.vec; ++q)
      for (int s2 = 0; s2 < args.p[q].nxy + (B == 8 ? args.p[q].nz : 0); ++s2)
        if (!make_rows_tmap(&args.lmap[q][s2], args.p[q].slot[s2], N / 16, 16, BF_BK * B / 16, 16)) {
          set_error("%s: cuTensorMapEncodeTiled (log) failed", what);
          return R3_ERR_CUDA;
        }
  }
  if (!make_rows_tmap(&args.pw4, pw, nblk, D, BF_BK, D)) {
    set_error("%s: cuTensorMapEncodeTiled failed", what);
    return R3_ERR_CUDA;
  }
  // K-chunks of <= BF_MAX_K blocks, a whole number of items per CTA of a
  // persistent grid (no partial second wave)
  const int per = B == 4 ? 1 : (B == 8 ? np : 2 * np + (args.nzs > 0 ? 1 : 0));   // items per K-chunk
  args.per = per;
  int64_t chunks = (nblk + BF_MAX_K - 1) / BF_MAX_K;
  int64_t items = chunks * per;
  items = (items + num_sms() - 1) / num_sms() * num_sms();
  chunks = (items + per - 1) / per;
  int64_t kc = (nblk + chunks - 1) / chunks;
  kc = (kc + BF_BK - 1) / BF_BK * BF_BK;
  items = (nblk + kc - 1) / kc * per;
  args.kc = kc;
  // every SM, items round-robin: CTA b takes items b, b + 148, ... whose
  // kinds (it % per) cycle because 148 % per != 0, so the cheap z items
  // spread over all CTAs (a grid of 147 = 21 x 7 gave 21 CTAs only z items)
  const unsigned grid = unsigned(items < num_sms() ? items : num_sms());
  ensure_smem(base_fold_tc_kernel<B, D>, BfLayout<B, D>::SMEM);
  base_fold_tc_kernel<B, D><<<grid, BF_THREADS, BfLayout<B, D>::SMEM, s>>>(args);
  return check_launch(what);
}

}  // namespace

// d = 64 form of r3_vfy_base_fold_q4 (same contract); -1 if not applicable.
int base_fold_q4_tc(int np, const int* nterms, const int64_t* coef, const uint64_t* const* xc,
                    const uint64_t* const* yc, const int* nz, const uint64_t* const* zc, const int64_t* zs,
                    int64_t N, const uint64_t* pw4, uint64_t* const* acc, uint64_t* const* zraw,
                    cudaStream_t s) {
  const int64_t nblk = (N + 3) / 4;
  if (nblk < 4096 || (uintptr_t(pw4) & 15)) return -1;
  return base_fold_tc_launch<4>(np, nterms, coef, xc, yc, nz, zc, zs, N, pw4, acc, zraw, s,
                                "r3_vfy_base_fold_q4(tc)");
}

namespace {

template <int B>
int base_fold_wide(int np, const int* nterms, const int64_t* coef, const uint64_t* const* xc,
                   const uint64_t* const* yc, const int* nz, const uint64_t* const* zc, const int64_t* zs,
                   int64_t N, const uint64_t* pw, int d, uint64_t* const* acc, uint64_t* const* zraw,
                   void* stream, const char* what) {
  if (np < 1 || np > 3 || (d != 64 && d != 16) || N < int64_t(B) * 4096 || (uintptr_t(pw) & 15) || !nterms || !nz) {
    set_error("%s: bad arguments (np %d, d %d, N %lld)", what, np, d, (long long)N);
    return R3_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  for (int q = 0; q < np; ++q) {
    if (nterms[q] < 1 || nterms[q] > 3 || nz[q] < 0 || nz[q] > 2 || zs[q] < 1) {
      set_error("%s: bad terms / z count for party %d", what, q);
      return R3_ERR_ARG;
    }
    if (cudaMemsetAsync(acc[q], 0, size_t(B) * B * d * 8, s) != cudaSuccess ||
        (nz[q] > 0 && cudaMemsetAsync(zraw[q], 0, size_t(nz[q]) * B * d * 8, s) != cudaSuccess)) {
      set_error("%s: memset failed", what);
      return R3_ERR_CUDA;
    }
  }
  return d == 64 ? base_fold_tc_launch<B, 64>(np, nterms, coef, xc, yc, nz, zc, zs, N, pw, acc, zraw, s, what)
                 : base_fold_tc_launch<B, 16>(np, nterms, coef, xc, yc, nz, zc, zs, N, pw, acc, zraw, s, what);
}

}  // namespace

extern "C" int r3_vfy_base_fold_q8(int np, const int* nterms, const int64_t* coef, const uint64_t* const* xc,
                                   const uint64_t* const* yc, const int* nz, const uint64_t* const* zc,
                                   const int64_t* zs, int64_t N, const uint64_t* pw8, int d,
                                   uint64_t* const* acc, uint64_t* const* zraw, void* stream) {
  return base_fold_wide<8>(np, nterms, coef, xc, yc, nz, zc, zs, N, pw8, d, acc, zraw, stream,
                           "r3_vfy_base_fold_q8");
}

extern "C" int r3_vfy_base_fold_q16(int np, const int* nterms, const int64_t* coef, const uint64_t* const* xc,
                                    const uint64_t* const* yc, const int* nz, const uint64_t* const* zc,
                                    const int64_t* zs, int64_t N, const uint64_t* pw16, int d,
                                    uint64_t* const* acc, uint64_t* const* zraw, void* stream) {
  return base_fold_wide<16>(np, nterms, coef, xc, yc, nz, zc, zs, N, pw16, d, acc, zraw, stream,
                            "r3_vfy_base_fold_q16");
}
