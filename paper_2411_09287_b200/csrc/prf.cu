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

#include "aes.cuh"

namespace r3 {

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

// Four-table kernels (aes.cuh) for bulk draws: one 1024-thread block per SM
// shares the 128 KB tables.
__global__ void __launch_bounds__(kAes4Threads, 1)
prf_ctr4_kernel(RoundKeys rk, u64 first, int64_t n, u64 mask, int mode, u64* __restrict__ out) {
  const Aes4Sel q = load_ttables4();
  const u64 b0 = first >> 1;
  const u64 nb = ((first + u64(n) + 1) >> 1) - b0;
  for (u64 t = blockIdx.x * u64(blockDim.x) + threadIdx.x; t < nb; t += u64(gridDim.x) * blockDim.x) {
    const u64 ctr = b0 + t;
    u64 lo, hi;
    aes4_ctr_words(rk, q, ctr, lo, hi);
    if (mode == 1) { lo &= 1ull; hi &= 1ull; } else { lo &= mask; hi &= mask; }
    const int64_t i0 = int64_t(2 * ctr - first);
    if (i0 >= 0 && i0 + 1 < n && (((uintptr_t)(out + i0)) & 15) == 0) {
      __stcs(reinterpret_cast<ulonglong2*>(out + i0), make_ulonglong2(lo, hi));
    } else {
      if (i0 >= 0 && i0 < n) out[i0] = lo;
      if (i0 + 1 >= 0 && i0 + 1 < n) out[i0 + 1] = hi;
    }
  }
}

__global__ void __launch_bounds__(kAes4Threads, 1)
prf_bits4_kernel(RoundKeys rk, u64 first, int nbits, int64_t lanes, u64* __restrict__ out) {
  const Aes4Sel q = load_ttables4();
  const bool paired = ((first | u64(lanes)) & 1) == 0;
  const int64_t units = paired ? lanes / 2 : lanes;
  for (int64_t u = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; u < units; u += int64_t(gridDim.x) * blockDim.x) {
    if (paired) {
      const int64_t l = 2 * u;
      u64 a0 = 0, a1 = 0;
      for (int j = 0; j < nbits; ++j) {
        const u64 w = first + u64(j) * u64(lanes) + u64(l);
        u32 blo, bhi;
        aes4_ctr_bit0s(rk, q, w >> 1, blo, bhi);
        a0 |= u64(blo) << j;
        a1 |= u64(bhi) << j;
      }
      *reinterpret_cast<ulonglong2*>(out + l) = make_ulonglong2(a0, a1);
    } else {
      u64 a = 0;
      for (int j = 0; j < nbits; ++j) {
        const u64 w = first + u64(j) * u64(lanes) + u64(u);
        u32 blo, bhi;
        aes4_ctr_bit0s(rk, q, w >> 1, blo, bhi);
        a |= u64((w & 1) ? bhi : blo) << j;
      }
      out[u] = a;
    }
  }
}

// Bulk draws (at least this many AES blocks) take the four-table kernels;
// smaller ones the single-table kernels (no 128 KB table fill per block).
constexpr int64_t kAes4MinBlocks = int64_t(1) << 16;

static bool aes4_init() {
  return ensure_smem(prf_ctr4_kernel, kAes4Smem) && ensure_smem(prf_bits4_kernel, kAes4Smem);
}

static unsigned aes4_grid(int64_t work) {
  const int64_t g = (work + kAes4Threads - 1) / kAes4Threads;
  return unsigned(g < num_sms() ? g : num_sms());
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
  imad_peak_kernel<<<num_sms() * 8, 256, 0, as_stream(stream)>>>(0x243f6a8885a308d3ull, iters, (u64*)sink);
  return check_launch("r3_imad_peak");
}

int r3::num_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  int v = __atomic_load_n(&cache[dev], __ATOMIC_RELAXED);
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    __atomic_store_n(&cache[dev], v, __ATOMIC_RELAXED);
  }
  return v;
}

bool r3::smem_attr_once(const void* func, int bytes) {
  // (kernel, device) -> bytes already granted; a handful of entries
  struct Entry { const void* f; int dev; int bytes; };
  static std::mutex mu;
  static Entry table[256];
  static int used = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < used; ++i)
    if (table[i].f == func && table[i].dev == dev && table[i].bytes >= bytes) return true;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (used < 256) table[used++] = {func, dev, bytes};
  return true;
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
  if (nblocks >= kAes4MinBlocks && aes4_init()) {
    prf_ctr4_kernel<<<aes4_grid(nblocks), kAes4Threads, kAes4Smem, as_stream(stream)>>>(
        k, first_u64, n, mask, mode, reinterpret_cast<u64*>(out));
    return check_launch("r3_prf_ctr");
  }
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
  if (units * nbits >= kAes4MinBlocks && aes4_init()) {
    prf_bits4_kernel<<<aes4_grid(units), kAes4Threads, kAes4Smem, as_stream(stream)>>>(
        k, first_u64, nbits, lanes, reinterpret_cast<u64*>(out));
    return check_launch("r3_prf_bits_packed");
  }
  prf_bits_packed_kernel<<<grid_for(units, kPrfThreads, 7), kPrfThreads, 0, as_stream(stream)>>>(
      k, first_u64, nbits, lanes, reinterpret_cast<u64*>(out));
  return check_launch("r3_prf_bits_packed");
}
