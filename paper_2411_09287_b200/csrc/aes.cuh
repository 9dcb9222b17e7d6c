// AES-128 counter-block helpers shared by the PRF kernels (prf.cu) and the
// fused bit-pipeline kernels (ripple.cu): one T-table (Te0) with the other
// three derived by byte rotation, replicated 32x in shared memory with
// column = lane so every lookup of a warp hits 32 distinct banks.
#pragma once

#include "r3_common.cuh"

namespace r3 {

#define R3_AES_SBOX { \
    0x63, 0x7c, 0x77, 0x7b, 0xf2, 0x6b, 0x6f, 0xc5, 0x30, 0x01, 0x67, 0x2b, 0xfe, 0xd7, 0xab, 0x76, \
    0xca, 0x82, 0xc9, 0x7d, 0xfa, 0x59, 0x47, 0xf0, 0xad, 0xd4, 0xa2, 0xaf, 0x9c, 0xa4, 0x72, 0xc0, \
    0xb7, 0xfd, 0x93, 0x26, 0x36, 0x3f, 0xf7, 0xcc, 0x34, 0xa5, 0xe5, 0xf1, 0x71, 0xd8, 0x31, 0x15, \
    0x04, 0xc7, 0x23, 0xc3, 0x18, 0x96, 0x05, 0x9a, 0x07, 0x12, 0x80, 0xe2, 0xeb, 0x27, 0xb2, 0x75, \
    0x09, 0x83, 0x2c, 0x1a, 0x1b, 0x6e, 0x5a, 0xa0, 0x52, 0x3b, 0xd6, 0xb3, 0x29, 0xe3, 0x2f, 0x84, \
    0x53, 0xd1, 0x00, 0xed, 0x20, 0xfc, 0xb1, 0x5b, 0x6a, 0xcb, 0xbe, 0x39, 0x4a, 0x4c, 0x58, 0xcf, \
    0xd0, 0xef, 0xaa, 0xfb, 0x43, 0x4d, 0x33, 0x85, 0x45, 0xf9, 0x02, 0x7f, 0x50, 0x3c, 0x9f, 0xa8, \
    0x51, 0xa3, 0x40, 0x8f, 0x92, 0x9d, 0x38, 0xf5, 0xbc, 0xb6, 0xda, 0x21, 0x10, 0xff, 0xf3, 0xd2, \
    0xcd, 0x0c, 0x13, 0xec, 0x5f, 0x97, 0x44, 0x17, 0xc4, 0xa7, 0x7e, 0x3d, 0x64, 0x5d, 0x19, 0x73, \
    0x60, 0x81, 0x4f, 0xdc, 0x22, 0x2a, 0x90, 0x88, 0x46, 0xee, 0xb8, 0x14, 0xde, 0x5e, 0x0b, 0xdb, \
    0xe0, 0x32, 0x3a, 0x0a, 0x49, 0x06, 0x24, 0x5c, 0xc2, 0xd3, 0xac, 0x62, 0x91, 0x95, 0xe4, 0x79, \
    0xe7, 0xc8, 0x37, 0x6d, 0x8d, 0xd5, 0x4e, 0xa9, 0x6c, 0x56, 0xf4, 0xea, 0x65, 0x7a, 0xae, 0x08, \
    0xba, 0x78, 0x25, 0x2e, 0x1c, 0xa6, 0xb4, 0xc6, 0xe8, 0xdd, 0x74, 0x1f, 0x4b, 0xbd, 0x8b, 0x8a, \
    0x70, 0x3e, 0xb5, 0x66, 0x48, 0x03, 0xf6, 0x0e, 0x61, 0x35, 0x57, 0xb9, 0x86, 0xc1, 0x1d, 0x9e, \
    0xe1, 0xf8, 0x98, 0x11, 0x69, 0xd9, 0x8e, 0x94, 0x9b, 0x1e, 0x87, 0xe9, 0xce, 0x55, 0x28, 0xdf, \
    0x8c, 0xa1, 0x89, 0x0d, 0xbf, 0xe6, 0x42, 0x68, 0x41, 0x99, 0x2d, 0x0f, 0xb0, 0x54, 0xbb, 0x16}
static const uint8_t kSbox[256] = R3_AES_SBOX;
static __device__ const uint8_t d_sbox[256] = R3_AES_SBOX;


struct RoundKeys {
  u32 w[44];
};

__device__ __forceinline__ u32 xtime8(u32 b) { return ((b << 1) ^ ((b & 0x80u) ? 0x1bu : 0u)) & 0xffu; }

// Te0[x] = (2s, s, s, 3s) from the most significant byte down.
__device__ __forceinline__ u32 te0_of(u32 s) {
  u32 s2 = xtime8(s);
  u32 s3 = s2 ^ s;
  return (s2 << 24) | (s << 16) | (s << 8) | s3;
}

__device__ __forceinline__ u32 bswap32(u32 x) { return __byte_perm(x, 0, 0x0123); }

constexpr int kPrfThreads = 256;

// AES-128 of the counter block BE128(ctr) with the per-lane replicated
// T-table Tl (= T + lane); returns the two little-endian keystream words.
__device__ __forceinline__ void aes_ctr_words(const RoundKeys& rk, const u32* Tl, u64 ctr, u64& lo, u64& hi) {
#define TE0(x) Tl[(x) << 5]
#define TE1(x) __funnelshift_r(TE0(x), TE0(x), 8)
#define TE2(x) __funnelshift_r(TE0(x), TE0(x), 16)
#define TE3(x) __funnelshift_r(TE0(x), TE0(x), 24)
#define SB(x) ((TE0(x) >> 8) & 0xffu)
  u32 s0 = rk.w[0];
  u32 s1 = rk.w[1];
  u32 s2 = u32(ctr >> 32) ^ rk.w[2];
  u32 s3 = u32(ctr) ^ rk.w[3];
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    u32 t0 = TE0(s0 >> 24) ^ TE1((s1 >> 16) & 0xff) ^ TE2((s2 >> 8) & 0xff) ^ TE3(s3 & 0xff) ^ rk.w[4 * r + 0];
    u32 t1 = TE0(s1 >> 24) ^ TE1((s2 >> 16) & 0xff) ^ TE2((s3 >> 8) & 0xff) ^ TE3(s0 & 0xff) ^ rk.w[4 * r + 1];
    u32 t2 = TE0(s2 >> 24) ^ TE1((s3 >> 16) & 0xff) ^ TE2((s0 >> 8) & 0xff) ^ TE3(s1 & 0xff) ^ rk.w[4 * r + 2];
    u32 t3 = TE0(s3 >> 24) ^ TE1((s0 >> 16) & 0xff) ^ TE2((s1 >> 8) & 0xff) ^ TE3(s2 & 0xff) ^ rk.w[4 * r + 3];
    s0 = t0; s1 = t1; s2 = t2; s3 = t3;
  }
  u32 o0 = (SB(s0 >> 24) << 24) ^ (SB((s1 >> 16) & 0xff) << 16) ^ (SB((s2 >> 8) & 0xff) << 8) ^ SB(s3 & 0xff) ^ rk.w[40];
  u32 o1 = (SB(s1 >> 24) << 24) ^ (SB((s2 >> 16) & 0xff) << 16) ^ (SB((s3 >> 8) & 0xff) << 8) ^ SB(s0 & 0xff) ^ rk.w[41];
  u32 o2 = (SB(s2 >> 24) << 24) ^ (SB((s3 >> 16) & 0xff) << 16) ^ (SB((s0 >> 8) & 0xff) << 8) ^ SB(s1 & 0xff) ^ rk.w[42];
  u32 o3 = (SB(s3 >> 24) << 24) ^ (SB((s0 >> 16) & 0xff) << 16) ^ (SB((s1 >> 8) & 0xff) << 8) ^ SB(s2 & 0xff) ^ rk.w[43];
#undef TE0
#undef TE1
#undef TE2
#undef TE3
#undef SB
  // keystream bytes are o0..o3 big-endian; u64 halves are little-endian reads
  lo = u64(bswap32(o0)) | (u64(bswap32(o1)) << 32);
  hi = u64(bswap32(o2)) | (u64(bswap32(o3)) << 32);
}

// ---------------------------------------------------------------------------
// Four-table form for the bulk PRF kernels.  128 KB of dynamic shared
// memory: region r (64 KB) holds Te(2r) and Te(2r+1); row x is 256 bytes,
// Te(2r)[x] replicated for the 32 lanes in bytes 0..127 (word = lane) and
// Te(2r+1)[x] in bytes 128..255.  With the tables 64 KB-aligned in the
// shared window, a lookup address base | (x << 8) | lane * 4 (| 128 for the
// odd table) is ONE byte permute of the state word: byte k of s to byte 1,
// the per-thread selector to bytes 0, 2 and 3 -- so a round is
// 16 PRMT + 16 LDS + 8 three-input XORs, with no rotates, masks or shifts
// (the single-table form spends about 100 instructions per round).  Every
// warp-wide lookup still hits 32 distinct banks.
// ---------------------------------------------------------------------------
constexpr int kAes4Bytes = 4 * 256 * 128;      // 128 KB of tables
constexpr int kAes4Smem = kAes4Bytes + 65536;  // + room to align them to 64 KB
constexpr int kAes4Threads = 1024;
extern __shared__ __align__(16) uint8_t aes4_smem[];

// Per-thread lookup selectors: the shared-window address of the tables is
// aligned to 64 KB, so its high half-word rides in bytes 2-3 of the PRMT
// operand and the permute yields the complete LDS address.
struct Aes4Sel {
  u32 y[4];   // table t: region base | (t & 1) * 128 | lane * 4
};

__device__ __forceinline__ Aes4Sel load_ttables4() {
  const u32 win = u32(__cvta_generic_to_shared(aes4_smem));
  const u32 base = (win + 65535u) & ~65535u;
  u32* W = reinterpret_cast<u32*>(aes4_smem + (base - win));
  for (int i = threadIdx.x; i < kAes4Bytes / 4; i += blockDim.x) {
    const int region = i >> 14, x = (i >> 6) & 255, col = i & 63;
    const int tbl = 2 * region + (col >> 5);
    const u32 t = te0_of(d_sbox[x]);
    W[i] = tbl ? __funnelshift_r(t, t, 8 * tbl) : t;
  }
  __syncthreads();
  Aes4Sel sel;
  const u32 lane4 = (threadIdx.x & 31) * 4;
#pragma unroll
  for (int t = 0; t < 4; ++t) sel.y[t] = base + 65536u * u32(t >> 1) + 128u * u32(t & 1) + lane4;
  return sel;
}

// Te(TBL)[byte BYTE of s]: one PRMT (s byte -> address byte 1, selector
// bytes 0, 2, 3) and one LDS.
template <int TBL, int BYTE>
__device__ __forceinline__ u32 t4(const Aes4Sel& q, u32 s) {
  const u32 a = __byte_perm(s, q.y[TBL], 0x7604 + 16 * BYTE);
  u32 v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// Rounds 1..9 of AES-128 on the counter block BE128(ctr); leaves the state
// before the final round in s0..s3.
__device__ __forceinline__ void aes4_rounds(const RoundKeys& rk, const Aes4Sel& q, u64 ctr, u32& s0, u32& s1,
                                            u32& s2, u32& s3) {
  s0 = rk.w[0];
  s1 = rk.w[1];
  s2 = u32(ctr >> 32) ^ rk.w[2];
  s3 = u32(ctr) ^ rk.w[3];
#pragma unroll
  for (int r = 1; r < 10; ++r) {
    const u32 t0 = t4<0, 3>(q, s0) ^ t4<1, 2>(q, s1) ^ t4<2, 1>(q, s2) ^ t4<3, 0>(q, s3) ^
                   rk.w[4 * r + 0];
    const u32 t1 = t4<0, 3>(q, s1) ^ t4<1, 2>(q, s2) ^ t4<2, 1>(q, s3) ^ t4<3, 0>(q, s0) ^
                   rk.w[4 * r + 1];
    const u32 t2 = t4<0, 3>(q, s2) ^ t4<1, 2>(q, s3) ^ t4<2, 1>(q, s0) ^ t4<3, 0>(q, s1) ^
                   rk.w[4 * r + 2];
    const u32 t3 = t4<0, 3>(q, s3) ^ t4<1, 2>(q, s0) ^ t4<2, 1>(q, s1) ^ t4<3, 0>(q, s2) ^
                   rk.w[4 * r + 3];
    s0 = t0; s1 = t1; s2 = t2; s3 = t3;
  }
}

// Final-round word: S-box bytes taken from the table whose byte lane holds s
// at that position (Te3: byte 3, Te0: byte 2, Te1: byte 1, Te2: byte 0).
__device__ __forceinline__ u32 aes4_last(const Aes4Sel& q, u32 a, u32 b, u32 c, u32 d, u32 k) {
  return (t4<3, 3>(q, a) & 0xff000000u) ^ (t4<0, 2>(q, b) & 0x00ff0000u) ^
         (t4<1, 1>(q, c) & 0x0000ff00u) ^ (t4<2, 0>(q, d) & 0x000000ffu) ^ k;
}

// The two little-endian keystream words of counter block ctr.
__device__ __forceinline__ void aes4_ctr_words(const RoundKeys& rk, const Aes4Sel& q, u64 ctr, u64& lo, u64& hi) {
  u32 s0, s1, s2, s3;
  aes4_rounds(rk, q, ctr, s0, s1, s2, s3);
  const u32 o0 = aes4_last(q, s0, s1, s2, s3, rk.w[40]);
  const u32 o1 = aes4_last(q, s1, s2, s3, s0, rk.w[41]);
  const u32 o2 = aes4_last(q, s2, s3, s0, s1, rk.w[42]);
  const u32 o3 = aes4_last(q, s3, s0, s1, s2, rk.w[43]);
  lo = u64(bswap32(o0)) | (u64(bswap32(o1)) << 32);
  hi = u64(bswap32(o2)) | (u64(bswap32(o3)) << 32);
}

// Bit 0 of both keystream words of block ctr (keystream bytes 0 and 8: the
// top bytes of final-round words 0 and 2 -- two S-box lookups).
__device__ __forceinline__ void aes4_ctr_bit0s(const RoundKeys& rk, const Aes4Sel& q, u64 ctr, u32& b_lo,
                                               u32& b_hi) {
  u32 s0, s1, s2, s3;
  aes4_rounds(rk, q, ctr, s0, s1, s2, s3);
  b_lo = ((t4<3, 3>(q, s0) ^ rk.w[40]) >> 24) & 1u;
  b_hi = ((t4<3, 3>(q, s2) ^ rk.w[42]) >> 24) & 1u;
}

__device__ __forceinline__ void load_ttable(u32* T) {
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) T[i] = te0_of(d_sbox[i >> 5]);
  __syncthreads();
}

}  // namespace r3
