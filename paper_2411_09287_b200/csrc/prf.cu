// AES-128-CTR keystream kernel: the PRF behind every Prg stream
// (reference prg.py:39-65: key = BLAKE2b(domain, key=pair seed) on the host,
// keystream = AES-128 over a zero IV with a big-endian 128-bit block counter,
// consumed 8 bytes at a time).
//
// Design (B200): one T-table (Te0) with the other three derived by byte
// rotation; the table is replicated 32x in shared memory, column = lane, so
// every lookup of a warp hits 32 distinct banks (conflict-free, one
// wavefront per LDS).  Each thread encrypts whole counter blocks and stores
// both 64-bit halves; the kernel is seekable (any first_u64), so party
// streams, shards and mid-block continuations cost nothing extra.
#include <cstdarg>
#include <atomic>
#include <cstring>

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
__device__ const uint8_t d_sbox[256] = R3_AES_SBOX;


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

__device__ __forceinline__ void load_ttable(u32* T) {
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) T[i] = te0_of(d_sbox[i >> 5]);
  __syncthreads();
}

__global__ void __launch_bounds__(kPrfThreads)
prf_ctr_kernel(RoundKeys rk, u64 first, int64_t n, u64 mask, int mode, u64* __restrict__ out) {
  // T[x*32 + lane] = Te0[x]: lane-private bank, conflict-free lookups.
  __shared__ u32 T[256 * 32];
  load_ttable(T);
  const u32* Tl = T + (threadIdx.x & 31);
  const u64 b0 = first >> 1;
  const u64 b_end = (first + u64(n) + 1) >> 1;
  const u64 nb = b_end - b0;
  for (u64 t = blockIdx.x * u64(blockDim.x) + threadIdx.x; t < nb; t += u64(gridDim.x) * blockDim.x) {
    const u64 ctr = b0 + t;
    u64 lo, hi;
    aes_ctr_words(rk, Tl, ctr, lo, hi);
    if (mode == 1) { lo &= 1ull; hi &= 1ull; } else { lo &= mask; hi &= mask; }
    const int64_t i0 = int64_t(2 * ctr - first);
    if (i0 >= 0 && i0 + 1 < n && (((uintptr_t)(out + i0)) & 15) == 0) {
      *reinterpret_cast<ulonglong2*>(out + i0) = make_ulonglong2(lo, hi);
    } else {
      if (i0 >= 0 && i0 < n) out[i0] = lo;
      if (i0 + 1 >= 0 && i0 + 1 < n) out[i0 + 1] = hi;
    }
  }
}

// Bit-packed draw_bits of an (nbits, lanes) matrix (gates.py:255-257,
// nonlinear.py:90-92): out[l] = sum_j (word(first + j*lanes + l) & 1) << j.
// When first and lanes are even one AES block serves lanes (2p, 2p+1).
__global__ void __launch_bounds__(kPrfThreads)
prf_bits_packed_kernel(RoundKeys rk, u64 first, int nbits, int64_t lanes, u64* __restrict__ out) {
  __shared__ u32 T[256 * 32];
  load_ttable(T);
  const u32* Tl = T + (threadIdx.x & 31);
  const bool paired = ((first | u64(lanes)) & 1) == 0;
  const int64_t units = paired ? lanes / 2 : lanes;
  for (int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u < units; u += int64_t(gridDim.x) * blockDim.x) {
    if (paired) {
      const int64_t l0 = 2 * u;
      u64 a0 = 0, a1 = 0;
      for (int j = 0; j < nbits; ++j) {
        const u64 w = first + u64(j) * u64(lanes) + u64(l0);
        u64 lo, hi;
        aes_ctr_words(rk, Tl, w >> 1, lo, hi);
        a0 |= (lo & 1ull) << j;
        a1 |= (hi & 1ull) << j;
      }
      *reinterpret_cast<ulonglong2*>(out + l0) = make_ulonglong2(a0, a1);
    } else {
      u64 a = 0;
      for (int j = 0; j < nbits; ++j) {
        const u64 w = first + u64(j) * u64(lanes) + u64(u);
        u64 lo, hi;
        aes_ctr_words(rk, Tl, w >> 1, lo, hi);
        a |= (((w & 1) ? hi : lo) & 1ull) << j;
      }
      out[u] = a;
    }
  }
}

}  // namespace r3

using namespace r3;

static thread_local char g_err[512];
static std::atomic<unsigned long long> g_launches{0};

void r3::count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" uint64_t r3_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

// Integer-ALU ceiling for the GR kernels: each thread runs 8 independent
// chains of 64-bit multiply-accumulates (the IMAD.WIDE + 2 IMAD sequence of
// every u64 MAC in gr.cu); `iters` MACs per chain.
__global__ void imad_peak_kernel(u64 seed, int iters, u64* __restrict__ sink) {
  u64 a[8], b = seed ^ (threadIdx.x * 0x9e3779b97f4a7c15ull), c = seed + blockIdx.x;
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = c + q;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = a[q] * b + c;
    b += 0x1234567ull;
  }
  u64 s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s ^= a[q];
  if (s == 0x5151515151ull) sink[0] = s;
}

extern "C" int r3_imad_peak(int iters, uint64_t* sink, void* stream) {
  imad_peak_kernel<<<kNumSMs * 8, 256, 0, as_stream(stream)>>>(0x243f6a8885a308d3ull, iters, (u64*)sink);
  return check_launch("r3_imad_peak");
}

void r3::set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" int r3_abi_version(void) { return R3_ABI_VERSION; }
extern "C" const char* r3_last_error(void) { return g_err; }

extern "C" void r3_aes128_expand(const uint8_t key[16], uint32_t rk[44]) {
  static const uint32_t rcon[10] = {0x01000000, 0x02000000, 0x04000000, 0x08000000, 0x10000000,
                                    0x20000000, 0x40000000, 0x80000000, 0x1b000000, 0x36000000};
  for (int i = 0; i < 4; ++i)
    rk[i] = (uint32_t(key[4 * i]) << 24) | (uint32_t(key[4 * i + 1]) << 16) |
            (uint32_t(key[4 * i + 2]) << 8) | uint32_t(key[4 * i + 3]);
  for (int i = 4; i < 44; ++i) {
    uint32_t t = rk[i - 1];
    if (i % 4 == 0) {
      t = (t << 8) | (t >> 24);
      t = (uint32_t(kSbox[t >> 24]) << 24) | (uint32_t(kSbox[(t >> 16) & 0xff]) << 16) |
          (uint32_t(kSbox[(t >> 8) & 0xff]) << 8) | uint32_t(kSbox[t & 0xff]);
      t ^= rcon[i / 4 - 1];
    }
    rk[i] = rk[i - 4] ^ t;
  }
}

extern "C" int r3_prf_ctr(const uint32_t rk[44], uint64_t first_u64, int64_t n, uint64_t mask, int mode,
                          uint64_t* out, void* stream) {
  if (n < 0 || (n > 0 && out == nullptr) || rk == nullptr || (mode != 0 && mode != 1)) {
    set_error("r3_prf_ctr: bad arguments");
    return R3_ERR_ARG;
  }
  if (n == 0) return R3_OK;
  RoundKeys k;
  memcpy(k.w, rk, sizeof(k.w));
  const int64_t nblocks = (int64_t((first_u64 + n + 1) >> 1) - int64_t(first_u64 >> 1));
  unsigned grid = grid_for(nblocks, kPrfThreads, 7);
  prf_ctr_kernel<<<grid, kPrfThreads, 0, as_stream(stream)>>>(k, first_u64, n, mask, mode,
                                                              reinterpret_cast<u64*>(out));
  return check_launch("r3_prf_ctr");
}

extern "C" int r3_prf_bits_packed(const uint32_t rk[44], uint64_t first_u64, int nbits, int64_t lanes,
                                  uint64_t* out, void* stream) {
  if (!rk || !out || nbits < 1 || nbits > 64 || lanes < 0) {
    set_error("r3_prf_bits_packed: bad arguments");
    return R3_ERR_ARG;
  }
  if (lanes == 0) return R3_OK;
  RoundKeys k;
  memcpy(k.w, rk, sizeof(k.w));
  const bool paired = ((first_u64 | uint64_t(lanes)) & 1) == 0;
  const int64_t units = paired ? lanes / 2 : lanes;
  prf_bits_packed_kernel<<<grid_for(units, kPrfThreads, 7), kPrfThreads, 0, as_stream(stream)>>>(
      k, first_u64, nbits, lanes, reinterpret_cast<u64*>(out));
  return check_launch("r3_prf_bits_packed");
}
