// tcgen05 / mbarrier / TMEM helpers shared by the tensor-core kernels
// (inline PTX for sm_100a; layouts per the canonical UMMA K-major no-swizzle
// form: 8-row x 16-byte core matrices).
#pragma once

#include <cuda.h>

#include "r3_common.cuh"

namespace r3 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no swizzle UMMA shared-memory descriptor (sm_100 version = 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE
}

// kind::i8 instruction descriptor: D s32, A/B uint8, both K-major.
__host__ __device__ constexpr uint32_t idesc_u8(int M, int N) {
  return (2u << 4) | (0u << 7) | (0u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_u8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 lanes x 16 columns of 32-bit words from TMEM (warp-collective).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
// 16 TMEM lanes x 8 columns (32-bit): thread t gets lane t/4 columns 2(t%4),
// 2(t%4)+1 in v[0..1] and lane t/4 + 8 in v[2..3] (the mma.sync C-fragment
// pattern), so 4 consecutive threads hold one row's 8 consecutive columns.
__device__ __forceinline__ void tmem_ld_16x256(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// byte i of each of x0..x3 (32-bit words) packed little-endian into one word
__device__ __forceinline__ uint32_t gather_byte(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, int i) {
  const uint32_t s01 = uint32_t(i) | (uint32_t(i + 4) << 4);  // (x0.byte i, x1.byte i)
  uint32_t lo = __byte_perm(x0, x1, s01);
  uint32_t hi = __byte_perm(x2, x3, s01);
  return __byte_perm(lo, hi, 0x5410);
}

// 4 x 4 byte transpose in 8 PRMT: o_j = (byte j of a, b, c, d)
__device__ __forceinline__ void bytes_t4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t& o0,
                                         uint32_t& o1, uint32_t& o2, uint32_t& o3) {
  const uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
  const uint32_t t2 = __byte_perm(c, d, 0x5140), t3 = __byte_perm(c, d, 0x7362);
  o0 = __byte_perm(t0, t2, 0x5410);
  o1 = __byte_perm(t0, t2, 0x7632);
  o2 = __byte_perm(t1, t3, 0x5410);
  o3 = __byte_perm(t1, t3, 0x7632);
}

// 16 u64 as 32 words (x[2q] low, x[2q+1] high half of word q) -> the 8
// byte-limb planes of those 16 values (plane i = byte i of each, 16 bytes)
__device__ __forceinline__ void split_limbs16(const uint32_t (&x)[32], uint4 (&out)[8]) {
  uint32_t o[8][4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    bytes_t4(x[8 * g + 0], x[8 * g + 2], x[8 * g + 4], x[8 * g + 6], o[0][g], o[1][g], o[2][g], o[3][g]);
    bytes_t4(x[8 * g + 1], x[8 * g + 3], x[8 * g + 5], x[8 * g + 7], o[4][g], o[5][g], o[6][g], o[7][g]);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) out[i] = make_uint4(o[i][0], o[i][1], o[i][2], o[i][3]);
}

__device__ __forceinline__ void split_limbs16(const u64 (&v)[16], uint4 (&out)[8]) {
  uint32_t w[32];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    w[2 * q] = uint32_t(v[q]);
    w[2 * q + 1] = uint32_t(v[q] >> 32);
  }
  split_limbs16(w, out);
}

// sum_s d[s] 2^(8 s) mod 2^64 for the 8 diagonal accumulators of one output,
// in 32-bit halves: diagonals 0-3 straddle the word boundary (one carry
// chain), diagonals 4-7 only reach the high word.
__device__ __forceinline__ uint64_t recombine8(const uint32_t d0, const uint32_t d1, const uint32_t d2,
                                               const uint32_t d3, const uint32_t d4, const uint32_t d5,
                                               const uint32_t d6, const uint32_t d7) {
  uint32_t lo, hi;
  asm("{\n\t"
      "add.cc.u32 %0, %2, %3;\n\t"
      "addc.u32 %1, %4, 0;\n\t"
      "add.cc.u32 %0, %0, %5;\n\t"
      "addc.u32 %1, %1, %6;\n\t"
      "add.cc.u32 %0, %0, %7;\n\t"
      "addc.u32 %1, %1, %8;\n\t"
      "}"
      : "=r"(lo), "=r"(hi)
      : "r"(d0), "r"(d1 << 8), "r"(d1 >> 24), "r"(d2 << 16), "r"(d2 >> 16), "r"(d3 << 24), "r"(d3 >> 8));
  hi += d4 + (d5 << 8) + (d6 << 16) + (d7 << 24);
  return (uint64_t(hi) << 32) | lo;
}

// core-matrix byte offset of (row, k) in a K-major no-swizzle tile with G row groups
__device__ __forceinline__ uint32_t core_off(int row, int k, int G) {
  return uint32_t((((k >> 4) * G + (row >> 3)) << 7) + ((row & 7) << 4) + (k & 15));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// 2-D TMA tile load (tensor map in kernel-parameter space) completing on bar.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// Host: tensor map over `rows` rows of `width` u64 (row stride rs_words,
// 16-byte aligned), box = 16 u64 x box_rows rows, 128-byte swizzle (16-byte
// chunk j of smem row r lands at chunk j ^ (r & 7)); rows past `rows` read
// as zero.
bool make_rows_tmap(CUtensorMap* map, const void* base, int64_t rows, int64_t rs_words, int box_rows,
                    int width = 64);

}  // namespace r3
