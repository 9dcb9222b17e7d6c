/*
 * r3b200.h -- C ABI of the B200 (sm_100a) kernels behind the ring3pc API.
 *
 * The reference (`ring3pc`, pure Python/numpy) has no FFI; its plugin seam is
 * the array-kernel layer `grvec` + `prg.Prg` plus the inline numpy in
 * gates/verify/nonlinear.  Each entry point below replaces one
 * of those numpy hot loops; the comment names the reference file:line it
 * stands in for.  Conventions:
 *
 *   - every array argument is a DEVICE pointer to uint64 words holding ring
 *     elements (Z_2^ell, ell <= 64; booleans as 0/1 words; GR(2^ell, d)
 *     elements as d consecutive words, constant coefficient first,
 *     grvec.py:1-7);
 *   - outputs are caller-allocated; no function allocates device memory;
 *   - `mask` = 2^ell - 1 is applied to every stored result (grvec.vmask);
 *   - `stream` is a cudaStream_t (NULL = legacy default stream);
 *   - return value 0 = success, otherwise an R3_ERR_* code with a message in
 *     r3_last_error() (thread-local).  Kernels are stateless and the only
 *     globals are const tables, so the library is reentrant across the
 *     three party threads (SURVEY.md 8b "Threading").
 */
#ifndef R3B200_H
#define R3B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define R3_OK 0
#define R3_ERR_ARG 1
#define R3_ERR_CUDA 2

#define R3_ABI_VERSION 1

/* Elementwise op codes for r3_ew. */
enum r3_ew_op {
  R3_EW_ADD = 0,  /* a + b                                                */
  R3_EW_SUB = 1,  /* a - b                                                */
  R3_EW_MUL = 2,  /* a * b                                                */
  R3_EW_AND = 3,  /* a & b                                                */
  R3_EW_XOR = 4,  /* a ^ b                                                */
  R3_EW_OR = 5,   /* a | b                                                */
  R3_EW_RSUB = 6, /* b - a                                                */
  R3_EW_COPY = 7  /* a (masked); b unused                                 */
};

/* Linear-combination operand: row i = sum_{q<nterms} coef[q] * p[q][i],
 * p[q] row-strided (rowstride in words; d coefficients contiguous), rows at
 * or beyond nvalid[q] read as zero. */
typedef struct r3_lin_operand {
  const uint64_t* p[4];
  int64_t rowstride[4];
  int64_t nvalid[4];
  uint64_t coef[4];
  int32_t nterms;
} r3_lin_operand;

int r3_abi_version(void);
const char* r3_last_error(void);
/* Number of kernels this library has launched in the process (bench
 * accounting of gpu_launches). */
uint64_t r3_launch_count(void);
/* Integer-ALU ceiling probe: 148*8 blocks x 256 threads x 8 chains x iters
 * dependent-free u64 multiply-adds (the u64 MAC of the GR kernels). */
int r3_imad_peak(int iters, uint64_t* sink, void* stream);

/* ---- PRF: AES-128-CTR streams (prg.py:39-65) ----------------------------
 * Host helper: FIPS-197 key expansion, 44 big-endian round-key words. */
void r3_aes128_expand(const uint8_t key[16], uint32_t rk[44]);
/* Keystream u64 number j (j = first_u64 .. first_u64+n-1) of AES-128-CTR with
 * a zero IV and 128-bit big-endian block counter: little-endian bytes
 * [8(j&1), 8(j&1)+8) of AES_K(BE128(j>>1)).  Replaces Prg.draw_u64 /
 * draw_base (mode 0: & mask) / draw_bits (mode 1: & 1), prg.py:50-62. */
int r3_prf_ctr(const uint32_t rk[44], uint64_t first_u64, int64_t n,
               uint64_t mask, int mode, uint64_t* out, void* stream);

/* Bit-packed draw_bits of an (nbits, lanes) bit matrix drawn row-major from
 * the stream at first_u64 (gates.py:255-257 / nonlinear.py:90-92):
 * out[l] = sum_j (keystream[first + j*lanes + l] & 1) << j.  The stream
 * advances by nbits*lanes words exactly as the reference's draw_bits. */
int r3_prf_bits_packed(const uint32_t rk[44], uint64_t first_u64, int nbits,
                       int64_t lanes, uint64_t* out, void* stream);

/* Fused a2b ripple MSB over Z_2 for the three simulated parties (replaces
 * the ell-2 sequential AND gates of nonlinear.py:133-160 with msb_only, each
 * a gates.py:52-117 Pi_mul).  rk01/rk02: round keys of the ("01","sha") and
 * ("02","sha") streams at u64 offsets o01/o02 (gate g draws out_s1, gamma_s1
 * from 01 at o01 + 2gL, o01 + (2g+1)L and out_s2 from 02 at o02 + gL).
 * eda[7]: (ell, lanes) edaBit rows (P0 s1, s2, total; P1 s1, m; P2 s2, m)
 * with row_stride words between rows; delta: the opened Delta per lane.
 * msb[7]: output MSB shares (same component order); msgs[3]: (ell-2, lanes)
 * payloads P0->P2 gamma share, P1 leg, P2 leg; logy/logz (optional, both or
 * neither): per-gate carry input and product output components. */
int r3_ripple_msb(const uint32_t rk01[44], const uint32_t rk02[44], uint64_t o01,
                  uint64_t o02, const uint64_t* delta, const uint64_t* const* eda,
                  int64_t row_stride, int ell, int64_t lanes, uint64_t* const* msb,
                  uint64_t* const* msgs, uint64_t* const* logy,
                  uint64_t* const* logz, void* stream);

/* ---- elementwise (grvec.py:18-40; sharing.py:95-230 linear ops) ----------
 * out[idx] = op(a[idx . a_strides], b[idx . b_strides]) over an ndim<=4 index
 * space `shape` (out contiguous).  Stride 0 broadcasts.  b == NULL uses the
 * scalar `imm` for b. */
int r3_ew(int op, int ndim, const int64_t* shape, uint64_t* out,
          const uint64_t* a, const int64_t* a_strides,
          const uint64_t* b, const int64_t* b_strides,
          uint64_t imm, uint64_t mask, void* stream);
/* Contiguous 1-d form of r3_ew (n words; b == NULL uses imm): the host's
 * hot elementwise call, no shape/stride arrays to marshal. */
int r3_ew_flat(int op, int64_t n, uint64_t* out, const uint64_t* a,
               const uint64_t* b, uint64_t imm, uint64_t mask, void* stream);
/* out = a - b - c (op 0) or a + b + c (op 1), & mask, contiguous n words:
 * opening a value from the three views (sharing.py:364-471) in one pass. */
int r3_ew3(int op, int64_t n, uint64_t* out, const uint64_t* a,
           const uint64_t* b, const uint64_t* c, uint64_t mask, void* stream);
/* k <= 4 contiguous length-n components in one launch: out[c] =
 * op(a[c], b ? b[c] : imm) & mask (the fields of one party's share view --
 * s1/s2/total/m, sharing.py:95-230 -- updated together).  Per-component
 * b may be NULL only if the whole b array is NULL. */
int r3_ew_multi(int op, int k, int64_t n, uint64_t* const* out,
                const uint64_t* const* a, const uint64_t* const* b,
                uint64_t imm, uint64_t mask, void* stream);
/* Sign-extending right shift on width-bit patterns (grvec.arith_rshift,
 * grvec.py:43-51); t in [0, width). */
int r3_ars(const uint64_t* a, int64_t n, int t, int width, uint64_t* out,
           void* stream);
/* out[j, l] = (a[l] >> j) & 1 for j < nbits (nonlinear.a2b public bits,
 * nonlinear.py:273). */
int r3_bit_planes(const uint64_t* a, int64_t lanes, int nbits, uint64_t* out,
                  void* stream);
/* *count += #{i : a[i] != b[i]} (b == NULL: #{a[i] != 0}).  Replaces the
 * SHA-256 digest comparison of Party.check_digest (runtime.py:115-124) and
 * the zero test of check_inner_product (verify.py:263).  count is a device
 * uint64 the caller zeroes. */
int r3_count_nonequal(const uint64_t* a, const uint64_t* b, int64_t n,
                      uint64_t* count, void* stream);
/* out[j] (+)= sum_i a[i*rowstride + j], i < n, j < inner (np.add.reduce over
 * axis 0: verify._sum_lanes verify.py:149-151, gates._sum_axis0). */
int r3_sum_axis0(const uint64_t* a, int64_t n, int64_t inner, int64_t rowstride,
                 uint64_t* out, uint64_t mask, int accumulate, void* stream);
/* out[l] = sum_i a[i,l] * b[i,l]   (P0's cross term, gates._pair_sum
 * gates.py:41-49, base ring).  Element (i,l) at p + i*rs + l*ls. */
int r3_dot_fold(int64_t n, int64_t lanes,
                const uint64_t* a, int64_t a_rs, int64_t a_ls,
                const uint64_t* b, int64_t b_rs, int64_t b_ls,
                uint64_t* out, uint64_t mask, void* stream);
/* Online Pi_dot leg of P1 (role 1) or P2 (role 2), base ring
 * (gates.dot_finish gates.py:92-106):
 *   P1: leg = g - sum_i mx*sy - sum_i my*sx
 *   P2: leg = sum_i mx*(my - sy) - sum_i my*sx + g
 * sx/sy are the party's mask halves. */
int r3_mul_leg(int role, int64_t n, int64_t lanes,
               const uint64_t* mx, int64_t mx_rs, int64_t mx_ls,
               const uint64_t* my, int64_t my_rs, int64_t my_ls,
               const uint64_t* sx, int64_t sx_rs, int64_t sx_ls,
               const uint64_t* sy, int64_t sy_rs, int64_t sy_ls,
               const uint64_t* g, uint64_t* out, uint64_t mask, void* stream);

/* ---- GR(2^ell, d) arithmetic (grvec.py:67-167; rings.py:180-241) -------
 * `lowterms` = bit mask of the exponents j < d with f_j = 1 (rings.py:180-188,
 * GrModulus.low_terms). */
/* out[i] = a[i] * b[i] in GR, rows broadcast when a_rs / b_rs == 0
 * (grvec.gr_mul grvec.py:78-93). */
int r3_gr_mul(const uint64_t* a, int64_t a_rs, const uint64_t* b, int64_t b_rs,
              uint64_t* out, int64_t rows, int d, uint64_t lowterms,
              uint64_t mask, void* stream);
/* out[f][row] = sum_{t<nterms} a[t*k + f][row] * c[t] in GR(2^ell, d):
 * k <= 4 fields (rows x d, contiguous), nterms <= 3 public single-element
 * weights -- the Lagrange recombination z' = h0 l0 + h1 l1 + h2 l2 of
 * Pi_rd (verify.py:233-236) for all of a party's fields in one launch. */
int r3_gr_lincomb(int k, int nterms, const uint64_t* const* a,
                  const uint64_t* const* c, uint64_t* const* out, int64_t rows,
                  int d, uint64_t lowterms, uint64_t mask, void* stream);
/* out[i] = s[i*s_stride] * g[i] (base scalar times GR element; the
 * reference's embedded-scalar gr_mul, identical values at d MACs/row). */
int r3_gr_scale_rows(const uint64_t* s, int64_t s_stride,
                     const uint64_t* g, int64_t g_rs, uint64_t* out,
                     int64_t rows, int d, uint64_t mask, void* stream);
/* Public per-level values of one Pi_rd reduction from the opened even point
 * ze (reference verify.py:215-241, grvec quad weights): out (4 x d) =
 * [l0, l1 - l0, l2, 1 - ze] with u = ze >> 1, l0 = (ze-1)(u-1), l1 = ze(2-ze),
 * l2 = u(ze-1) in GR(2^width, d) (mask = 2^width - 1); if Mo and Mz are both
 * non-NULL also the (d x d) multiplication matrices of 1 - ze and ze.  One
 * launch replaces the ~15 small GR operations of the reference's helper. */
int r3_gr_quad(const uint64_t* ze, int d, uint64_t lowterms, uint64_t mask,
               uint64_t* out, uint64_t* Mo, uint64_t* Mz, void* stream);
/* M (d x d): row j = x^j * c mod f, so that (a * c) = a_row . M. */
int r3_gr_mulmat(const uint64_t* c, int d, uint64_t lowterms, uint64_t* M,
                 void* stream);
/* out[i] = A[i] . M (+ C[i])   -- multiplication of many GR elements by one
 * element whose matrix is M; A and C are lin-operands (line evaluation
 * verify.py:239-240 as f0 + (f1 - f0)*zeta, gr_powers block doubling
 * grvec.py:130-141, scale_gr by a public element). */
int r3_gr_matmul(r3_lin_operand A, const uint64_t* M, int has_c,
                 r3_lin_operand C, uint64_t* out, int64_t rows, int d,
                 uint64_t mask, void* stream);
/* Pipelined tensor-core contraction for d = 64:
 *   out[r] = P0[r] . M0 + P1[r] . M1      (P1 == NULL: out[r] = P0[r] . M0)
 * P0/P1 rows at p + r*rs (16-byte aligned), rows >= nv read as zero.  The
 * line evaluation f0 + (f1 - f0) zeta is f0 . M_{1-zeta} + f1 . M_zeta. */
int r3_gr_matmul2_tc(const uint64_t* p0, int64_t rs0, int64_t nv0,
                     const uint64_t* p1, int64_t rs1, int64_t nv1,
                     const uint64_t* M0, const uint64_t* M1, uint64_t* out,
                     int64_t rows, uint64_t mask, void* stream);
/* Several r3_gr_matmul2_tc jobs sharing M0 / M1 in one launch (the line
 * evaluations of every component a party reduces at one level,
 * verify.py:239-240): job j is out_j[r] = P0_j[r] . M0 + P1_j[r] . M1 for
 * r < rows[j], both operands present with >= 1 valid row; 1..8 jobs. */
int r3_gr_matmul2_tc_multi(int njobs, const uint64_t* const* p0, const int64_t* rs0,
                           const int64_t* nv0, const uint64_t* const* p1, const int64_t* rs1,
                           const int64_t* nv1, const uint64_t* M0, const uint64_t* M1,
                           uint64_t* const* outs, const int64_t* rows, uint64_t mask,
                           void* stream);
/* d = 16 form of r3_gr_matmul2_tc_multi (rows of 16 coefficients). */
int r3_gr_matmul2_tc16_multi(int njobs, const uint64_t* const* p0, const int64_t* rs0,
                             const int64_t* nv0, const uint64_t* const* p1, const int64_t* rs1,
                             const int64_t* nv1, const uint64_t* M0, const uint64_t* M1,
                             uint64_t* const* outs, const int64_t* rows, uint64_t mask,
                             void* stream);
/* One operand times q <= 4 public GR(2^64, 64) multiplication matrices in
 * one pass: outs[k][r] = p[r] . Ms[k] for r < rows (rows of 64 u64 at
 * stride rs words, 16-byte aligned).  The four level-2 tables of a
 * verification (r^(4j) . C_a, verify.py:215-241 applied from the base log)
 * come from one read of the r^(4j) table. */
int r3_gr_matmul_q_tc(const uint64_t* p, int64_t rs, int64_t rows,
                      const uint64_t* const* Ms, uint64_t* const* outs, int q,
                      uint64_t mask, void* stream);

/* out[j] = sum_{a < 16} p[16 j + a] K[a] (K: 16 x 64 words, p: rows x 16
 * words, 16-byte aligned) as a K = 16 byte-limb GEMM on the tensor cores:
 * the level-4 y-side rows kappa_a y_(16j + a) of a multiplication log with
 * blocks of sixteen (verify.py:237-240 applied four times from the base
 * log; the arithmetic of r3_vfy_line_b_const with B = 16, d = 64). */
int r3_gr_matmul_k16_tc(const uint64_t* p, int64_t rows, const uint64_t* K,
                        uint64_t* out, uint64_t mask, void* stream);

/* out[c] = (a[c] + b[c] - 2 p[c]) & mask for k <= 4 same-length components
 * (the fields of one share view): the arithmetic XOR of bit shares,
 * a + b - 2ab (nonlinear.py:43-55), in one pass. */
/* out[c][l] = sum_{i < rows} w[i] (a[c][i L + l] + b[c][i L + l]) & mask,
 * k <= 4 components of (rows, L) arrays, rows <= 64: the linear part of the
 * edaBits recomposition sum_i 2^i (m_i + r'_i) (nonlinear.py:104-118). */
int r3_wsum_rows(int k, int rows, int64_t L, uint64_t* const* out, const uint64_t* const* a,
                 const uint64_t* const* b, const uint64_t* w, uint64_t mask, void* stream);
/* out[c][i L + l] = w[i] a[c][i L + l] & mask, k <= 4 components of (rows, L)
 * arrays: a public per-row scaling of every field of a share view (the
 * -2^(i+1) x side of the edaBits inner product, nonlinear.py:104-118). */
int r3_scale_rows(int k, int rows, int64_t L, uint64_t* const* out, const uint64_t* const* a,
                  const uint64_t* w, uint64_t mask, void* stream);
int r3_xor_arith(int k, int64_t n, uint64_t* const* out, const uint64_t* const* a,
                 const uint64_t* const* b, const uint64_t* const* p, uint64_t mask, void* stream);

/* Dot logs (n, L) with n % 16 == 0 at d = 16 (the edaBits inner products,
 * verify.py:182-241): the first four reductions from the base log.
 * r3_vfy_lane16_fold: acc[a*16 + b] = sum_l pw[l] sum_{blocks j of lane l}
 * sum_t coef[t] x_t[16j + a] y_t[16j + b] (256 x d words, zeroed here);
 * element i of lane l at i*L + l.  r3_vfy_lane16_line: the level-4 rows
 * (row l*(n/16) + j) sum_a kappa[a] x[16j + a], times pw[l] in GR(2^64, d)
 * when pow_side (f = t^d + sum of the lowterms monomials). */
/* Level-4 rows of a d = 16 multiplication log with blocks of sixteen
 * straight from the base shares (verify.py:237-240 applied four times):
 * row j = sum_a coef[a] x[16j + a] (coef: 16 x 16 words), times pw16[j] in
 * GR(2^64, 16) when pow_side (x side: coef[a] = r^a kappa_a; y side:
 * kappa_a).  Replaces the sixteen N/16-row tables. */
int r3_vfy_mul16_line(int pow_side, int ncomp, const uint64_t* const* xc, int64_t N,
                      const uint64_t* pw16, const uint64_t* coef, uint64_t lowterms, int d,
                      uint64_t* const* out, uint64_t mask, void* stream);
int r3_vfy_lane16_fold(int nterms, const int64_t* coef, const uint64_t* const* xc,
                       const uint64_t* const* yc, int64_t L, int64_t n,
                       const uint64_t* pw, int d, uint64_t* acc, void* stream);
int r3_vfy_lane16_line(int pow_side, int ncomp, const uint64_t* const* xc, int64_t L,
                       int64_t n, const uint64_t* pw, const uint64_t* kappa,
                       uint64_t lowterms, int d, uint64_t* const* out, uint64_t mask,
                       void* stream);

/* Dense-level leg folds for d = 16 of up to four leg terms (several
 * simulated parties) in one tensor-core pass: term k (x, y' = c0 y0 + c1 y1,
 * (N, 16) row-major, y1 may be null) adds its h(1) = sum o_x (x) o_y' and
 * h(2) = sum t_x (x) t_y' (t = 2 odd - even over row pairs) into the 31
 * unreduced words acc1[party[k]] / acc2[party[k]] (zeroed here; parties
 * without terms may pass null).  Same values as r3_vfy_level_fold per role
 * (verify.py:229-231 via gates.py:92-106). */
int r3_vfy_level_fold16_tc(int nterms, const int* party, const uint64_t* const* xs,
                           const uint64_t* const* y0s, const uint64_t* const* y1s,
                           const int64_t* c0, const int64_t* c1, int64_t N,
                           uint64_t* const* acc1, uint64_t* const* acc2, void* stream);

/* d = 16 form of r3_gr_matmul2_tc (rows of 16 coefficients, M0/M1 16 x 16):
 * both operands K-concatenate into one 32-byte kind::i8 K-step. */
int r3_gr_matmul2_tc16(const uint64_t* p0, int64_t rs0, int64_t nv0,
                     const uint64_t* p1, int64_t rs1, int64_t nv1,
                     const uint64_t* M0, const uint64_t* M1, uint64_t* out,
                     int64_t rows, uint64_t mask, void* stream);
/* acc[0..2d-2] += unreduced polynomial sum_i F[i] (x) G[i] (the inner
 * products of reduce_dimension / check_inner_product, verify.py:154-161,
 * gates.dot_finish.fold over GR). acc must be zeroed by the caller before the
 * first term. */
int r3_gr_dotsum(r3_lin_operand F, r3_lin_operand G, int64_t rows, int d,
                 uint64_t* acc, void* stream);
/* out[0..d-1] (+)= acc reduced mod f and masked. */
int r3_gr_reduce_poly(const uint64_t* acc, int d, uint64_t lowterms,
                      uint64_t* out, uint64_t mask, int accumulate,
                      void* stream);
/* nrows reductions in one launch: row i of acc (2d - 1 words, consecutive)
 * reduced mod f and masked into out[i*d .. i*d + d - 1] (the h(1) / h(2)
 * folds of a level, verify.py:229-231). */
int r3_gr_reduce_poly_rows(const uint64_t* acc, int nrows, int d, uint64_t lowterms,
                           uint64_t* out, uint64_t mask, void* stream);

/* ---- share-domain matmul on the tensor cores (ppml.py:412-427 algebra) ----
 * Operand preparation: value = c0*P0 + c1*P1 (P1 may be NULL) split into 8
 * byte-limb planes laid out as UMMA-ready tiles.
 *   A: rows x K row-major  -> [rows/128][K/32][8][128x32]   (32 KB per tile)
 *   B: K x cols row-major  -> [cols/64][K/32][8][64x32]      (16 KB per tile)
 * rows % 128 == 0, cols % 64 == 0, K % 32 == 0. */
int r3_limb_tiles_a(const uint64_t* p0, uint64_t c0, const uint64_t* p1,
                    uint64_t c1, int64_t rows, int64_t K, uint8_t* dst,
                    void* stream);
int r3_limb_tiles_b(const uint64_t* p0, uint64_t c0, const uint64_t* p1,
                    uint64_t c1, int64_t K, int64_t cols, uint8_t* dst,
                    void* stream);
/* out = addend (+ or, sub != 0, -) sum_p A_p . B_p  mod 2^64 (masked), M x N
 * row-major; up to 3 K-concatenated (A, B) tile pairs, total K <= 16384
 * (exact 32-bit diagonal accumulation).  addend may be NULL. */
int r3_u64_gemm_tc(int npairs, const uint8_t* const* a_tiles,
                   const uint8_t* const* b_tiles, const int64_t* K, int64_t M,
                   int64_t N, const uint64_t* addend, int sub, uint64_t* out,
                   uint64_t mask, void* stream);

/* ---- fused verification stages (verify.py:168-241) ----------------------
 * Compressed triples are never materialised (SURVEY.md finding 5): x'_i =
 * pw[i/n] * x_i (x a base share, pw the challenge powers r^k), y'_i = y_i
 * lifted.  Element i of a base component lives at c + (i % n)*ks + (i / n)*ls
 * (n = 1 for multiplication logs; n = dot length for Pi_bsv lane-major
 * consolidation, verify.py:195-201).
 *
 * r3_vfy_powsum: out[c] = sum_l comps[c][l] * pw[l] for c < ncomp
 * (z compression, verify.py:178 and 204). */
int r3_vfy_powsum(int ncomp, const uint64_t* const* comps, int64_t stride,
                  int64_t lanes, const uint64_t* pw, int d, uint64_t* out,
                  uint64_t mask, void* stream);
/* Level-1 h(1)/h(2) folds of one party (verify.py:220-231) on compressed
 * operands.  Terms t < nterms: coef[t] * fold(x-comp xi[t], y-comp yi[t]);
 * out_h1/out_h2 (d words each) receive the sums. */
int r3_vfy_l1_fold(int nterms, const int64_t* coef, const uint64_t* const* xc,
                   const uint64_t* const* yc, int64_t N, int64_t n,
                   int64_t ks, int64_t ls, const uint64_t* pw, int d,
                   uint64_t* out_h1, uint64_t* out_h2, uint64_t mask,
                   void* stream);
/* One party's h(1) and h(2) leg folds of a dense reduction level in one pass
 * (verify.py:223-230 with gates.py:100-106): rows of dense (N, d) component
 * arrays, pairs (2j, 2j+1), zero pad for odd N.  role 0: xa/ya = x/y total;
 * role 1: xa/ya = m, xb/yb = s1; role 2: m and s2.  acc1/acc2 (2d-1 words
 * each, zeroed by the caller) receive the unreduced polynomial sums. */
int r3_vfy_level_fold(int role, const uint64_t* xa, const uint64_t* xb,
                      const uint64_t* ya, const uint64_t* yb, int64_t N, int d,
                      uint64_t* acc1, uint64_t* acc2, void* stream);
/* Level-1 line evaluation of x components (verify.py:239):
 * out[c][j] = X_c[2j] * A[(2j)/tq] + X_c[2j+1] * B[(2j+1)/tq] with public
 * tables A = pw(1-ze), B = pw ze (tq = 2 with A/B over even/odd powers for
 * multiplication logs; tq = n with A/B over all powers for dot logs);
 * X_c[N] reads as 0 when N is odd. */
int r3_vfy_l1_line_x(int ncomp, const uint64_t* const* xc, int64_t N,
                     int64_t n, int64_t ks, int64_t ls, const uint64_t* A,
                     const uint64_t* B, int64_t tq, int d,
                     uint64_t* const* out, uint64_t mask, void* stream);
/* Level-1 line evaluation of y components (verify.py:240):
 * out[c][j] = Y_c[2j] * a + Y_c[2j+1] * b with public a = 1-ze, b = ze. */
int r3_vfy_l1_line_y(int ncomp, const uint64_t* const* yc, int64_t N,
                     int64_t n, int64_t ks, int64_t ls, const uint64_t* a,
                     const uint64_t* b, int d, uint64_t* const* out,
                     uint64_t mask, void* stream);

/* One pass over the power table for a multiplication log (n = 1, base
 * components contiguous): the z power sum of r3_vfy_powsum (nz <= 2
 * components, stride zs, masked), the 16 level-2 accumulators of
 * r3_vfy_l2_fold (acc, 16 x d, unmasked) and the level-1 folds of
 * r3_vfy_l1_fold derived from them (h1, h2, masked) -- verify.py:168-179
 * + 215-241 at k = 0, 1.  Same terms/coefficients as r3_vfy_l2_fold. */
int r3_vfy_base_fold(int nterms, const int64_t* coef,
                     const uint64_t* const* xc, const uint64_t* const* yc,
                     int nz, const uint64_t* const* zc, int64_t zs, int64_t N,
                     const uint64_t* pw, int d, uint64_t* acc, uint64_t* h1,
                     uint64_t* h2, uint64_t* zsum, uint64_t mask, void* stream);
/* r3_vfy_base_fold for np <= 3 parties in ONE pass over the power table
 * (party q's operands at xc/yc[3q + t], zc[2q + c], coef[3q + t]; outputs
 * acc/h1/h2/zsum[q]).  Blocks of the np parties on the same table rows are
 * adjacent, so the table streams from HBM once. */
/* Base fold against the table pw4[j] = r^(4j) (one row per block of four
 * elements): raw accumulators acc'[a*4+b] = sum_j s^{ab}_j r^(4j) (16 x d)
 * and zraw[c*4+a] = sum_j z_c[4j+a] r^(4j); the caller multiplies by r^a
 * and derives the level-1 folds with r3_vfy_base_fold_finish. */
int r3_vfy_base_fold_q4(int np, const int* nterms, const int64_t* coef,
                        const uint64_t* const* xc, const uint64_t* const* yc,
                        const int* nz, const uint64_t* const* zc, const int64_t* zs,
                        int64_t N, const uint64_t* pw4, int d, uint64_t* const* acc,
                        uint64_t* const* zraw, void* stream);
/* Base fold over blocks of eight against pw8[j] = r^(8j) (d = 64 or 16, N >= 8 *
 * 4096, tensor cores): acc'[a*8+b] = sum_j s^{ab}_j r^(8j) (64 x d) and
 * zraw[c*8+a] = sum_j z_c[8j+a] r^(8j) -- every accumulator the first THREE
 * reductions need (verify.py:215-241 at k = 0, 1, 2); same operand
 * conventions as r3_vfy_base_fold_q4. */
int r3_vfy_base_fold_q8(int np, const int* nterms, const int64_t* coef,
                        const uint64_t* const* xc, const uint64_t* const* yc,
                        const int* nz, const uint64_t* const* zc, const int64_t* zs,
                        int64_t N, const uint64_t* pw8, int d, uint64_t* const* acc,
                        uint64_t* const* zraw, void* stream);
/* The same over blocks of sixteen against pw16[j] = r^(16j) (N >= 16 * 4096):
 * acc'[a*16+b] (256 x d) and zraw[c*16+a] -- the accumulators of the first
 * FOUR reductions. */
int r3_vfy_base_fold_q16(int np, const int* nterms, const int64_t* coef,
                         const uint64_t* const* xc, const uint64_t* const* yc,
                         const int* nz, const uint64_t* const* zc, const int64_t* zs,
                         int64_t N, const uint64_t* pw16, int d, uint64_t* const* acc,
                         uint64_t* const* zraw, void* stream);
/* h1/h2 level-1 folds from the 16 accumulators; masks the nz z sums. */
int r3_vfy_base_fold_finish(int d, int nz, const uint64_t* acc, uint64_t* h1,
                            uint64_t* h2, uint64_t* zsum, uint64_t mask, void* stream);
int r3_vfy_base_fold_multi(int np, const int* nterms, const int64_t* coef,
                           const uint64_t* const* xc, const uint64_t* const* yc,
                           const int* nz, const uint64_t* const* zc,
                           const int64_t* zs, int64_t N, const uint64_t* pw, int d,
                           uint64_t* const* acc, uint64_t* const* h1,
                           uint64_t* const* h2, uint64_t* const* zsum,
                           uint64_t mask, void* stream);
/* Second reduction straight from the base log (vfy2.cu): for blocks of four
 * elements 4j+a, acc[(a*4+b)] = sum_j s^{ab}_j pw[(4j+a)/n] with the party's
 * scalar leg products s^{ab}_j = sum_t coef_t x_t[4j+a] y_t[4j+b]; 16 x d
 * words, zeroed here.  The caller applies the 16 public line weights. */
int r3_vfy_l2_fold(int nterms, const int64_t* coef, const uint64_t* const* xc,
                   const uint64_t* const* yc, int64_t N, int64_t n, int64_t ks,
                   int64_t ls, const uint64_t* pw, int d, uint64_t* acc,
                   void* stream);
/* out_c[j] = sum_{a<B} X_c[Bj+a] * T_a[(Bj+a)/tq] with tables T_a at
 * tabs + a*tab_stride (words), B <= 16 (B > 4: multiplication logs, n = 1,
 * tq = B, ncomp <= 4): level-log2(B) vectors from the base log. */
int r3_vfy_line_b(int B, int ncomp, const uint64_t* const* xc, int64_t N,
                  int64_t n, int64_t ks, int64_t ls, const uint64_t* tabs,
                  int64_t tab_stride, int64_t tq, int d, uint64_t* const* out,
                  uint64_t mask, void* stream);
/* out_c[j] = sum_{b<B} Y_c[Bj+b] * g_b (B <= 16 public GR constants; B > 4
 * for n = 1 and ncomp <= 4 only). */
int r3_vfy_line_b_const(int B, int ncomp, const uint64_t* const* yc, int64_t N,
                        int64_t n, int64_t ks, int64_t ls, const uint64_t* g,
                        int d, uint64_t* const* out, uint64_t mask,
                        void* stream);

/* r3_vfy_level_fold of all three simulated parties in ONE launch (d = 64,
 * tensor cores; honest sessions where P1 and P2 hold the same m): vectors
 * tx / ty (P0's sums), mx / my (m), s1x / s1y (P1), s2x / s2y (P2), each N
 * rows of 64 words; acc1[r] / acc2[r] (127 words each, zeroed here) receive
 * party r's unreduced h(1) / h(2) folds.  The items of a K chunk are
 * adjacent, so m is read from HBM about once for both of its parties. */
int r3_vfy_level_fold_joint(const uint64_t* tx, const uint64_t* ty, const uint64_t* mx,
                            const uint64_t* my, const uint64_t* s1x, const uint64_t* s1y,
                            const uint64_t* s2x, const uint64_t* s2y, int64_t N,
                            uint64_t* const* acc1, uint64_t* const* acc2, void* stream);

/* The local arithmetic of one verification reduction round for all three
 * simulated parties (gates.py:52-177 for the h(1) / h(2) vfy.dot gates of
 * single GR elements, sharing.py:364-420 for the opened even point 2 zeta):
 * F0/F1/F2 the parties' two folds (2 x d each, contiguous rows), d01 the
 * 01-stream draws (om1.s1, g1.s1, om2.s1, g2.s1), d02 the 02-stream draws
 * (om1.s2, om2.s2), zs1 / zs2 / zm zeta's shares; out (14 x d): om_tot[2],
 * Gamma - s1 [2], leg1[2], leg2[2], m[2], 2 zeta.s1, 2 zeta.s2, 2 zeta.m,
 * ze = 2 zeta. */
int r3_vfy_round(int d, const uint64_t* F0, const uint64_t* F1, const uint64_t* F2,
                 const uint64_t* d01, const uint64_t* d02, const uint64_t* zs1,
                 const uint64_t* zs2, const uint64_t* zm, uint64_t* out, uint64_t mask,
                 void* stream);

/* ---- packed GF(2^d) verification of boolean multiplication logs ----
 * Over the boolean ring the verification ring is GR(2, d) = GF(2^d) (d <= 32);
 * the reference multiplies its (n, d) 0/1 words on bit-packed words
 * (grvec.py:96-115).  Level vectors here are packed from the start: one
 * uint32 per element, bit k = coefficient of x^k.  f_low = the modulus f
 * without x^d (rings.py:180-188).  r, ze: (1, d) 0/1 words in device memory
 * (the opened challenge r and the opened even point ze = 2 zeta).  Party leg
 * terms are nterms component-index pairs (tx[t], ty[t]); their +-1
 * coefficients are 1 mod 2.  Folds come back unpacked, (rows, d) 0/1 words.
 * scratch: 8 uint32 of device memory per call in flight.
 *
 * Level 0 straight from the base log (verify.py:168-179 fused with the first
 * reduction's inner products, verify.py:229-231): h1 = sum over odd i of
 * r^i t_i, h2 = sum over even i (char 2: f2 = 2 f1 - f0 = f0), t_i = the xor
 * of the leg bit products x_tx[i] y_ty[i]; zsum_c = sum_i r^i z_c[i].
 * folds: (2 + nz) rows h1, h2, zsum_0, zsum_1. */
int r3_gfv_base_fold(int ncomp, const uint64_t* const* x, const uint64_t* const* y,
                     int nterms, const int* tx, const int* ty, int nz,
                     const uint64_t* const* z, int64_t N, const uint64_t* r,
                     int d, uint32_t f_low, uint64_t* folds, uint32_t* scratch,
                     void* stream);
/* One line evaluation out_j = f0_j + (f1_j - f0_j) ze (verify.py:239-240,
 * odd n_in padded with a zero row, verify.py:220-222) of every component,
 * from the base bits and the powers r^i (src_base: x'_i = r^i x_i,
 * y'_i = y_i) or from packed uint32 rows (16-byte aligned), fused with the
 * h(1)/h(2) folds of the output level (folds != NULL: 2 rows).  Outputs:
 * ceil(n_in / 2) packed uint32 rows, or (rows, d) 0/1 words if unpacked. */
int r3_gfv_line(int src_base, int ncomp, const void* const* x, const void* const* y,
                int64_t n_in, const uint64_t* r, const uint64_t* ze, int d,
                uint32_t f_low, int unpacked, void* const* ox, void* const* oy,
                int nterms, const int* tx, const int* ty, uint64_t* folds,
                uint32_t* scratch, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* R3B200_H */
