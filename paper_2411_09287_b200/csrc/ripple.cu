// Fused secure comparison core: the ripple-carry MSB of a2b for all three
// simulated parties in one pass (reference nonlinear.py:133-160 with
// msb_only, called from a2b nonlinear.py:267-274 and drelu_online).
//
// Per lane the reference runs ell - 2 sequential boolean AND gates (Pi_mul
// over Z_2 via dot_prepare / dot_finish, gates.py:52-117) on the carry
//     c_{j+1} = b_j c_j + a_j (b_j + c_j),     sum_{ell-1} = a + b + c
// where a = bit j of the opened Delta (public) and b_j the edaBit shares.
// Gate g (bit j = g + 1) draws, in stream order, the output mask
// (P0: "01" then "02", sha_random) and P0's Gamma share s1 ("01", sha_input):
//     01 stream: out_s1 at o01 + 2g L + l, gamma_s1 at o01 + (2g+1) L + l
//     02 stream: out_s2 at o02 + g L + l
// (L lanes, l this lane).  Everything is over Z_2: add = xor, mul = and.
// The kernel evaluates P0, P1 and P2 of every gate in registers, one thread
// per lane (AES-128-CTR keystream words computed in place from the same
// per-lane T-table the PRF kernel uses), and writes what the protocol
// exposes: the three message payloads of every gate (P0 -> P2 Gamma share,
// P1 <-> P2 legs), the MSB share of each party and, optionally, the gate-log
// operands (carry in, product out) for the batch verification.
#include "aes.cuh"

namespace r3 {

struct RippleIn {
  const u64* p0_s1;   // edaBit shares, (ell, lanes) rows of 0/1 words
  const u64* p0_s2;
  const u64* p0_tot;
  const u64* p1_s1;
  const u64* p1_m;
  const u64* p2_s2;
  const u64* p2_m;
  int64_t row_stride;
};

struct RippleOut {
  u64* msb[7];        // P0 s1, s2, total; P1 s1, m; P2 s2, m   (lanes)
  u64* msg[3];        // (ell - 2, lanes): P0 gamma s2, P1 leg1, P2 leg2
  u64* logy[7];       // optional (ell - 2, lanes): carry into gate g, same component order
  u64* logz[7];       // optional: gate output (mask comps, m_z for P1 / P2)
};

// bit 0 of stream word idx (four-table AES, aes.cuh)
__device__ __forceinline__ u64 ks_bit(const RoundKeys& rk, const Aes4Sel& q, u64 idx) {
  u32 blo, bhi;
  aes4_ctr_bit0s(rk, q, idx >> 1, blo, bhi);
  return (idx & 1) ? bhi : blo;
}

constexpr int kRippleThreads = 768;   // 24 warps: the carry state needs ~80 registers

__global__ void __launch_bounds__(kRippleThreads, 1)
ripple_msb_kernel(RoundKeys rk01, RoundKeys rk02, u64 o01, u64 o02, const u64* __restrict__ delta, RippleIn in,
                  RippleOut out, int ell, int64_t lanes, int write_log) {
  const Aes4Sel Tl = load_ttables4();
  const int64_t rs = in.row_stride;
  const int ng = ell - 2;
  for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < lanes; l += int64_t(gridDim.x) * blockDim.x) {
    const u64 dv = delta[l];
    // carry after bit 0: b_0 * a_0
    u64 a = dv & 1ull;
    u64 c[7] = {in.p0_s1[l] & a, in.p0_s2[l] & a, in.p0_tot[l] & a, in.p1_s1[l] & a, in.p1_m[l] & a,
                in.p2_s2[l] & a, in.p2_m[l] & a};
    for (int j = 1; j < ell; ++j) {
      a = (dv >> j) & 1ull;
      const int64_t off = j * rs + l;
      const u64 b[7] = {in.p0_s1[off], in.p0_s2[off], in.p0_tot[off], in.p1_s1[off], in.p1_m[off],
                        in.p2_s2[off], in.p2_m[off]};
      u64 bc[7];
#pragma unroll
      for (int q = 0; q < 7; ++q) bc[q] = b[q] ^ c[q];
      if (j == ell - 1) {
        // sum = (b + c) + a: the public bit enters m only (P1, P2)
        bc[4] ^= a;
        bc[6] ^= a;
#pragma unroll
        for (int q = 0; q < 7; ++q) out.msb[q][l] = bc[q];
        break;
      }
      const int g = j - 1;
      const u64 out_s1 = ks_bit(rk01, Tl, o01 + u64(2 * g) * u64(lanes) + u64(l));
      const u64 gam_s1 = ks_bit(rk01, Tl, o01 + u64(2 * g + 1) * u64(lanes) + u64(l));
      const u64 out_s2 = ks_bit(rk02, Tl, o02 + u64(g) * u64(lanes) + u64(l));
      const u64 rz_tot = out_s1 ^ out_s2;
      // P0: Gamma = x y + r_z on its mask totals, dealt as (gamma_s1, gamma_s2)
      const u64 gam2 = ((b[2] & c[2]) ^ rz_tot) ^ gam_s1;
      // P1 leg: Gamma_1 - m_x s_y1 - m_y s_x1;  P2 leg: m_x m_y + Gamma_2 - m_x s_y2 - m_y s_x2
      const u64 leg1 = gam_s1 ^ (b[4] & c[3]) ^ (c[4] & b[3]);
      const u64 leg2 = (b[6] & c[6]) ^ gam2 ^ (b[6] & c[5]) ^ (c[6] & b[5]);
      const u64 mz = leg1 ^ leg2;
      const int64_t mo = int64_t(g) * lanes + l;
      out.msg[0][mo] = gam2;
      out.msg[1][mo] = leg1;
      out.msg[2][mo] = leg2;
      const u64 z[7] = {out_s1, out_s2, rz_tot, out_s1, mz, out_s2, mz};
      if (write_log) {
#pragma unroll
        for (int q = 0; q < 7; ++q) {
          out.logy[q][mo] = c[q];
          out.logz[q][mo] = z[q];
        }
      }
      // carry = x y + a (b + c)
#pragma unroll
      for (int q = 0; q < 7; ++q) c[q] = z[q] ^ (bc[q] & a);
    }
  }
  (void)ng;
}

}  // namespace r3

using namespace r3;

extern "C" int r3_ripple_msb(const uint32_t* rk01, const uint32_t* rk02, uint64_t o01, uint64_t o02,
                             const uint64_t* delta, const uint64_t* const* eda, int64_t row_stride, int ell,
                             int64_t lanes, uint64_t* const* msb, uint64_t* const* msgs, uint64_t* const* logy,
                             uint64_t* const* logz, void* stream) {
  if (!rk01 || !rk02 || !delta || !eda || !msb || !msgs || ell < 2 || ell > 64 || lanes < 0 || row_stride < lanes) {
    set_error("r3_ripple_msb: bad arguments");
    return R3_ERR_ARG;
  }
  if (lanes == 0) return R3_OK;
  RoundKeys k01, k02;
  for (int i = 0; i < 44; ++i) {
    k01.w[i] = rk01[i];
    k02.w[i] = rk02[i];
  }
  RippleIn in{reinterpret_cast<const u64*>(eda[0]), reinterpret_cast<const u64*>(eda[1]),
              reinterpret_cast<const u64*>(eda[2]), reinterpret_cast<const u64*>(eda[3]),
              reinterpret_cast<const u64*>(eda[4]), reinterpret_cast<const u64*>(eda[5]),
              reinterpret_cast<const u64*>(eda[6]), row_stride};
  RippleOut out{};
  const int write_log = (logy && logz) ? 1 : 0;
  for (int q = 0; q < 7; ++q) {
    out.msb[q] = reinterpret_cast<u64*>(msb[q]);
    if (write_log) {
      out.logy[q] = reinterpret_cast<u64*>(logy[q]);
      out.logz[q] = reinterpret_cast<u64*>(logz[q]);
    }
  }
  for (int q = 0; q < 3; ++q) out.msg[q] = reinterpret_cast<u64*>(msgs[q]);
  if (!ensure_smem(ripple_msb_kernel, kAes4Smem)) {
    set_error("r3_ripple_msb: cannot reserve %d bytes of shared memory", kAes4Smem);
    return R3_ERR_CUDA;
  }
  const int64_t blocks = (lanes + kRippleThreads - 1) / kRippleThreads;
  const unsigned grid = unsigned(blocks < num_sms() ? blocks : num_sms());
  ripple_msb_kernel<<<grid, kRippleThreads, kAes4Smem, as_stream(stream)>>>(k01, k02, o01, o02,
                                                                 reinterpret_cast<const u64*>(delta), in, out,
                                                                 ell, lanes, write_log);
  return check_launch("r3_ripple_msb");
}
