// bc_device.cuh -- device-side building blocks of the Bicoptor 2.0 hot path
// (sm_100a).  Integer-only: no tensor cores, nothing here is a contraction.
//
// Per element j (global index) the computing parties run Alg 7 steps 1-8
// (P:875-888), P2 runs steps 9-10 and P0/P1 step 11;
// ReLU (Alg 8) adds the Beaver combine.  The randomness is a
// ChaCha keystream per (seed, label), addressed by global element index
// (DESIGN.md "PRG tape"), generated in registers and never stored.
#pragma once
#include <cstdint>

namespace bc {

// ---------------------------------------------------------------------------
// Stream labels: 8 ASCII bytes read little-endian (ChaCha state words 14-15).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr uint64_t lbl(const char (&s)[9]) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | (uint64_t)(uint8_t)s[i];
  return v;
}
constexpr uint64_t L_TAPEA = lbl("bc2.tpa1");  // seed01, 16 B / element (compact tape, part A)
constexpr uint64_t L_TAPEB = lbl("bc2.tpb1");  // seed01,  8 B / element (compact tape, part B)
constexpr uint64_t L_TAPEP = lbl("bc2.tpp1");  // seed01, 32 B / element (pair tape: p <= 131, 28-bit (r, rho) draws)
constexpr uint64_t L_FB = lbl("bc2.fb01");     // seed01, fallback, counter j*256+k
constexpr uint64_t L_RESP = lbl("bc2.resp");   // seed02, [DReLU']_0
constexpr uint64_t L_A02 = lbl("bc2.ta02");    // seed02, [a]_0
constexpr uint64_t L_B02 = lbl("bc2.tb02");    // seed02, [b]_0
constexpr uint64_t L_C02 = lbl("bc2.tc02");    // seed02, [c]_0
constexpr uint64_t L_A12 = lbl("bc2.ta12");    // seed12, [a]_1
constexpr uint64_t L_B12 = lbl("bc2.tb12");    // seed12, [b]_1

constexpr uint32_t PERM_LIMIT_8 = 53261u * 40320u;  // largest multiple of 8! below 2^31
constexpr uint32_t RHO_WORD_LIMIT = 253u * 257u * 257u * 257u;  // largest multiple of 257^3 below 2^32

struct Key {
  uint32_t k[8];
  uint32_t m7;  // = 2^7, read from the kernel parameter bank so ptxas cannot strength-reduce
                // rotl_fma's multiplies back into ALU shifts (LEA.HI / SHF)
};

// Kernel-side protocol constants (derived on the host from bc_params).
struct KP {
  uint64_t ymask;      // 2^ell - 1
  uint32_t f, w, p, S, lx;
  uint32_t fsh, fhi;   // f & 31, f >= 32 (window extraction)
  uint32_t wmask;      // 2^w - 1
  uint32_t perm_lim;   // floor(2^31 / S!) * S!
  uint32_t fact;       // S!
  // pair tape: d = (p-1) p, one 28-bit draw per slot, u / d = umulhi(u, pair_mag) >> pair_sh for u < 2^28
  uint32_t pair_d, pair_lim, pair_mag, pair_sh;  // d, floor(2^28 / d) d, ceil(2^(32+k) / d), k = floor(log2 d)
  // magic multipliers of the runtime divisions (exact for the ranges used):
  uint32_t mag_p, mag_q;   // ceil(2^32 / p), ceil(2^32 / (p-1)): x / d = umulhi(x, mag) for x < 2^16
  uint32_t mag_f, sh_f;    // ceil(2^(31+l) / S!), l - 1 (l = ceil(log2 S!)): x / S! = umulhi(x, mag_f) >> sh_f, x < 2^31
  uint32_t one;            // = 1, opaque to ptxas (add_fma: a * one + b stays an IMAD on the FMA pipe)
};

// The compact literal domain is one fixed parameter set (w = lx = 7, p = 131, 8 slots): its
// kernels overwrite the runtime fields with literals so that every mod-p step compiles to
// constants.  make_kp derives the same values on the host; the literal parity tests cover both.
__device__ __forceinline__ KP kp_literal(const KP& kp) {
  KP k = kp;
  k.w = 7u; k.lx = 7u; k.p = 131u; k.S = 8u; k.wmask = 127u;
  k.fact = 40320u; k.perm_lim = 53261u * 40320u;
  k.pair_d = 130u * 131u; k.pair_lim = 15762u * 17030u;
  k.pair_mag = (uint32_t)(((1ull << 46) + 17029ull) / 17030ull); k.pair_sh = 14u;
  k.mag_p = (uint32_t)(((1ull << 32) + 130ull) / 131ull);
  k.mag_q = (uint32_t)(((1ull << 32) + 129ull) / 130ull);
  k.mag_f = (uint32_t)(((1ull << 47) + 40319ull) / 40320ull);  // l = ceil(log2 8!) = 16
  k.sh_f = 15u;
  return k;
}

// ---------------------------------------------------------------------------
// ChaCha_R block (RFC 8439 sec. 2.3), words 12-13 = 64-bit counter, 14-15 =
// 64-bit label.  The key lives in the constant bank.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t rotl(uint32_t v, int n) { return __funnelshift_l(v, v, n); }

// rotl on the FMA pipe: (x << n) + (x >> (32-n)) = lo(x * 2^n) + hi(x * 2^n),
// one IMAD.SHL and one IMAD.HI with addend.  ChaCha is xor/rotate heavy (ALU
// pipe: LOP3, SHF) and add light (FMA pipe: IMAD.IADD); moving one of the four
// rotations of each quarter round to the FMA pipe balances the two pipes.
__device__ __forceinline__ uint32_t rotl_fma(uint32_t v, uint32_t two_n) { return __umulhi(v, two_n) + v * two_n; }

// BC_ROT_FMA = how many of the 8 quarter rounds of a double round take their
// rotate-by-7 on the FMA pipe (IMAD + IMAD.HI = 3 FMA issue slots, measured:
// IMAD.HI runs at half rate) instead of the ALU pipe (SHF).  ChaCha is ALU
// bound (xor + rotate), so moving a few rotates to the idle FMA pipe helps
// until the FMA pipe saturates (tools/variants.py).
#ifndef BC_ROT_FMA
#define BC_ROT_FMA 0
#endif
#define BC_QR_ALU(a, b, c, d)      \
  a += b; d ^= a; d = rotl(d, 16); \
  c += d; b ^= c; b = rotl(b, 12); \
  a += b; d ^= a; d = rotl(d, 8);  \
  c += d; b ^= c; b = rotl(b, 7);
#define BC_QR_FMA(a, b, c, d)      \
  a += b; d ^= a; d = rotl(d, 16); \
  c += d; b ^= c; b = rotl(b, 12); \
  a += b; d ^= a; d = rotl(d, 8);  \
  c += d; b ^= c; b = rotl_fma(b, key.m7);
#define BC_QR_SEL(i, a, b, c, d) \
  if ((i) < BC_ROT_FMA) { BC_QR_FMA(a, b, c, d) } else { BC_QR_ALU(a, b, c, d) }

// Double rounds are kept (mostly) rolled: a full R = 20 unroll is ~1000
// instructions per call site and the fused kernel's call sites then overflow
// the instruction cache (ncu: "no_instruction" was the top stall).
#ifndef BC_CHACHA_UNROLL
#define BC_CHACHA_UNROLL 1
#endif
constexpr int kChachaUnroll = BC_CHACHA_UNROLL;

template <int R>
__device__ __forceinline__ void chacha(const Key& key, uint64_t ctr, uint64_t label, uint32_t (&o)[16]) {
  uint32_t x0 = 0x61707865u, x1 = 0x3320646eu, x2 = 0x79622d32u, x3 = 0x6b206574u;
  uint32_t x4 = key.k[0], x5 = key.k[1], x6 = key.k[2], x7 = key.k[3];
  uint32_t x8 = key.k[4], x9 = key.k[5], x10 = key.k[6], x11 = key.k[7];
  const uint32_t c0 = (uint32_t)ctr, c1 = (uint32_t)(ctr >> 32);
  const uint32_t l0 = (uint32_t)label, l1 = (uint32_t)(label >> 32);
  uint32_t x12 = c0, x13 = c1, x14 = l0, x15 = l1;
#pragma unroll kChachaUnroll
  for (int r = 0; r < R; r += 2) {
    BC_QR_SEL(0, x0, x4, x8, x12) BC_QR_SEL(2, x1, x5, x9, x13) BC_QR_SEL(4, x2, x6, x10, x14)
    BC_QR_SEL(6, x3, x7, x11, x15) BC_QR_SEL(1, x0, x5, x10, x15) BC_QR_SEL(3, x1, x6, x11, x12)
    BC_QR_SEL(5, x2, x7, x8, x13) BC_QR_SEL(7, x3, x4, x9, x14)
  }
  o[0] = x0 + 0x61707865u; o[1] = x1 + 0x3320646eu; o[2] = x2 + 0x79622d32u; o[3] = x3 + 0x6b206574u;
  o[4] = x4 + key.k[0]; o[5] = x5 + key.k[1]; o[6] = x6 + key.k[2]; o[7] = x7 + key.k[3];
  o[8] = x8 + key.k[4]; o[9] = x9 + key.k[5]; o[10] = x10 + key.k[6]; o[11] = x11 + key.k[7];
  o[12] = x12 + c0; o[13] = x13 + c1; o[14] = x14 + l0; o[15] = x15 + l1;
}

// A (key, label) pair with the two column quarter rounds of the first round
// that involve neither counter word already applied (columns 2 and 3: words
// 2, 6, 10, 14 and 3, 7, 11, 15 are constants, key and label).  Computed on
// the host per (seed, stream label); the kernel reads it from the parameter
// bank, so the first round costs two quarter rounds instead of four.
struct KeyPre {
  uint32_t k[8];
  uint32_t l0, l1;
  uint32_t c[8];  // x2, x6, x10, x14, x3, x7, x11, x15 after the first column round
  uint32_t c1[4]; // x1, x5, x9, x13 after it when the counter's high word x13 is 0 (chacha_pre<R, true>)
};

// HI0: every counter of the launch is below 2^32 (chosen on the host from elem_base + n), so
// column 1 of the first round (x1, x5, x9, x13 = 0) is precomputed too: one quarter round left.
template <int R, bool HI0 = false, int UNR = kChachaUnroll>
__device__ __forceinline__ void chacha_pre(const KeyPre& P, uint64_t ctr, uint32_t (&o)[16]) {
  uint32_t x0 = 0x61707865u, x1 = 0x3320646eu;
  uint32_t x4 = P.k[0], x5 = P.k[1], x8 = P.k[4], x9 = P.k[5];
  const uint32_t c0 = (uint32_t)ctr, c1 = HI0 ? 0u : (uint32_t)(ctr >> 32);
  uint32_t x12 = c0, x13 = c1;
  if (HI0) {
    x1 = P.c1[0]; x5 = P.c1[1]; x9 = P.c1[2]; x13 = P.c1[3];
    BC_QR_ALU(x0, x4, x8, x12)
  } else {
    BC_QR_ALU(x0, x4, x8, x12) BC_QR_ALU(x1, x5, x9, x13)
  }
  uint32_t x2 = P.c[0], x6 = P.c[1], x10 = P.c[2], x14 = P.c[3];
  uint32_t x3 = P.c[4], x7 = P.c[5], x11 = P.c[6], x15 = P.c[7];
  BC_QR_ALU(x0, x5, x10, x15) BC_QR_ALU(x1, x6, x11, x12) BC_QR_ALU(x2, x7, x8, x13) BC_QR_ALU(x3, x4, x9, x14)
#pragma unroll UNR
  for (int r = 2; r < R; r += 2) {
    BC_QR_ALU(x0, x4, x8, x12) BC_QR_ALU(x1, x5, x9, x13) BC_QR_ALU(x2, x6, x10, x14) BC_QR_ALU(x3, x7, x11, x15)
    BC_QR_ALU(x0, x5, x10, x15) BC_QR_ALU(x1, x6, x11, x12) BC_QR_ALU(x2, x7, x8, x13) BC_QR_ALU(x3, x4, x9, x14)
  }
  o[0] = x0 + 0x61707865u; o[1] = x1 + 0x3320646eu; o[2] = x2 + 0x79622d32u; o[3] = x3 + 0x6b206574u;
  o[4] = x4 + P.k[0]; o[5] = x5 + P.k[1]; o[6] = x6 + P.k[2]; o[7] = x7 + P.k[3];
  o[8] = x8 + P.k[4]; o[9] = x9 + P.k[5]; o[10] = x10 + P.k[6]; o[11] = x11 + P.k[7];
  o[12] = x12 + c0; o[13] = x13 + c1; o[14] = x14 + P.l0; o[15] = x15 + P.l1;
}

// ---------------------------------------------------------------------------
// Small helpers
// ---------------------------------------------------------------------------
// x mod 257 for any 32-bit x: floor(x/257) = floor(x * (2^40+1)/257 / 2^40).
__device__ __forceinline__ uint32_t mod257(uint32_t x) {
  const uint32_t q = __umulhi(x, 0xFF00FF01u) >> 8;
  return x - q * 257u;
}
// Zero-extended byte m (0..3) of v.
__device__ __forceinline__ uint32_t byte_of(uint32_t v, int m) { return __byte_perm(v, 0u, 0x4440u | (uint32_t)m); }

// Fisher-Yates over S slots on a nibble array (reading C9): for m = S-1..1,
// k_m = q mod (m+1), q /= (m+1), swap nibbles m and k_m.  Nibble m of the
// result is the pre-shuffle slot that lands in slot m (a PRMT selector).
template <int S>
__device__ __forceinline__ uint32_t perm_sel(uint32_t q) {
  uint32_t sel = 0x76543210u;
#pragma unroll
  for (int m = S - 1; m >= 1; --m) {
    const uint32_t k = q % (uint32_t)(m + 1);
    q /= (uint32_t)(m + 1);
    const uint32_t a = (sel >> (4 * m)) & 15u, b = (sel >> (4 * k)) & 15u, d = a ^ b;
    sel ^= (d << (4 * m)) | (d << (4 * k));
  }
  return sel;
}

__device__ __forceinline__ uint32_t perm_sel_rt(uint32_t q, uint32_t S) {
  uint32_t sel = 0x76543210u;
#pragma unroll
  for (int m = 7; m >= 1; --m) {
    if ((uint32_t)m < S) {
      const uint32_t k = q % (uint32_t)(m + 1);
      q /= (uint32_t)(m + 1);
      const uint32_t a = (sel >> (4 * m)) & 15u, b = (sel >> (4 * k)) & 15u, d = a ^ b;
      sel ^= (d << (4 * m)) | (d << (4 * k));
    }
  }
  return sel;
}

// ---------------------------------------------------------------------------
// Rejection fallback (reading C10): sequential u32 words of
// ChaCha(seed01, L_FB, counter j*256 + k).  Rare (~1e-4 per element); kept
// out of line so the fast path carries no extra block.
// ---------------------------------------------------------------------------
template <int R>
struct FbStream {
  Key key;
  uint64_t j;
  uint32_t blk[16];
  uint32_t pos, kc;
  __device__ uint32_t next() {
    if (pos == 16) {
      chacha<R>(key, j * 256u + kc, L_FB, blk);
      ++kc;
      pos = 0;
    }
    return blk[pos++];
  }
};

struct Draws {  // raw draws of one element: perm index, 8 mask u16, 8 reshare u16
  uint32_t idx;
  uint32_t um[8];
  uint32_t ur[8];
};

template <int R>
__device__ __noinline__ void fallback(Draws& d, uint64_t j, Key key, uint32_t S, uint32_t perm_lim,
                                      uint32_t mask_lim /*0: masks never rejected*/, uint32_t rho_lim,
                                      uint32_t dmask /*draw width: 2^28 - 1 for the pair tape*/) {
  FbStream<R> fb;
  fb.key = key; fb.j = j; fb.pos = 16; fb.kc = 0;
  if (d.idx >= perm_lim) {
    uint32_t v = fb.next() & 0x7FFFFFFFu;
    while (v >= perm_lim) v = fb.next() & 0x7FFFFFFFu;
    d.idx = v;
  }
  if (mask_lim) {
    for (uint32_t m = 0; m < S; ++m)
      if (d.um[m] >= mask_lim) {
        uint32_t v = fb.next() & dmask;
        while (v >= mask_lim) v = fb.next() & dmask;
        d.um[m] = v;
      }
  }
  for (uint32_t m = 0; m < S; ++m)
    if (d.ur[m] >= rho_lim) {
      uint32_t v = fb.next() & dmask;
      while (v >= rho_lim) v = fb.next() & dmask;
      d.ur[m] = v;
    }
}
template <int R>
__device__ __noinline__ void fallback(Draws& d, uint64_t j, const Key* key, uint32_t S, uint32_t perm_lim,
                                      uint32_t mask_lim, uint32_t rho_lim, uint32_t dmask) {
  fallback<R>(d, j, *key, S, perm_lim, mask_lim, rho_lim, dmask);  // key by address (__grid_constant__ params)
}

// ---------------------------------------------------------------------------
// Decoded seed01 randomness of one element (Alg 7 steps 1, 6, 7, 8).
// ---------------------------------------------------------------------------
// Wide-tape (generic p, slots) randomness of one element.
struct Tape {
  uint32_t t;        // blinding bit (step 1)
  uint32_t sel;      // permutation as a PRMT nibble selector (step 6)
  uint32_t r[8];     // r_m in Z_p^* (step 7)
  uint32_t rho[8];   // reshare rho_m in Z_p (step 8)
};

// Pair tape (every lx <= 7 domain but the compact one: p <= 131, 3..8 slots): 32 B per element,
// two elements per block (label bc2.tpp1); T[0..7] = keystream bytes [32 j, 32 j + 32).
//   T0: t | perm index (reject >= floor(2^31/S!) S!)
//   T1..T7 as one 224-bit little-endian D: u_m = (D >> 28 m) & (2^28 - 1), one draw per slot m < S,
//   reject u >= floor(2^28/d) d (d = (p-1) p); x = u mod d, r_m = 1 + x mod (p-1), rho_m = x div (p-1).
// The fallback stream yields low-28-bit draws (fallback() with the reshare loop disabled).  The
// compact literal kernels (p = 131, 8 slots) pass kp_literal(kp), so the same code compiles to constants.
template <int R>
__device__ __forceinline__ void decode_pair(const uint32_t* T, uint64_t j, const Key& k01, const KP& kp, Tape& tp) {
  Draws d;
  tp.t = T[0] >> 31;
  d.idx = T[0] & 0x7FFFFFFFu;
  bool bad = d.idx >= kp.perm_lim;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int bit = 28 * m, w = bit >> 5, sh = bit & 31;
    const uint32_t nxt = w < 6 ? T[2 + w] : 0u;
    d.um[m] = __funnelshift_r(T[1 + w], nxt, sh) & 0x0FFFFFFFu;
    d.ur[m] = 0u;
    bad |= ((uint32_t)m < kp.S) & (d.um[m] >= kp.pair_lim);
  }
  if (__builtin_expect(bad, 0)) {
    Draws f = d;
    fallback<R>(f, j, k01, kp.S, kp.perm_lim, kp.pair_lim, 1u, 0x0FFFFFFFu);
    d = f;
  }
  const uint32_t q1 = kp.p - 1u;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t x = d.um[m] - kp.pair_d * (__umulhi(d.um[m], kp.pair_mag) >> kp.pair_sh);
    const uint32_t q = __umulhi(x, kp.mag_q);  // x div (p-1), exact for x < 2^16
    tp.r[m] = 1u + x - q1 * q;
    tp.rho[m] = q;
  }
  tp.sel = perm_sel_rt(d.idx - kp.fact * (__umulhi(d.idx, kp.mag_f) >> kp.sh_f), kp.S);
}

// ---------------------------------------------------------------------------
// Alg 7 steps 1-8 for one party: W_m, the message to P2 (values in Z_p).
//   1-2 s = (-1)^t x;  P1 works on n = -s (Alg 5, reading C3)
//   3   u_i = window [f+i, f+i+w) (Alg 5, k1 = f+i, k2 = ell-w-f-i)
//   4   v_i = u_i + u_{i+1} - 1 (P0 carries the -1), v_lx = u_lx - 1
//   5   modulo switch (Alg 6) -> encoded as bytes v'-1
//   6   shuffle: PRMT with the permutation selector
//   7-8 W_m = v'_m r_m + rho_m (P0) / v'_m r_m - rho_m (P1)  mod p
// ---------------------------------------------------------------------------
// x mod p for x < 2^24 by the host's magic (KP::mag_p = ceil(2^32 / p), p <= 257): exact.
__device__ __forceinline__ uint32_t modp_small(uint32_t x, const KP& kp) {
  return x - kp.p * __umulhi(x, kp.mag_p);
}

template <int PARTY>
__device__ __forceinline__ void party_W_rt(uint64_t x, const KP& kp, const Tape& tp, uint32_t (&W)[8]) {
  const uint64_t nx = 0ull - x;
  const uint64_t v = (PARTY == 0) ? (tp.t ? nx : x) : (tp.t ? x : nx);
  const uint32_t win = (uint32_t)(v >> kp.f);
  uint32_t u[9];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t a = (win >> i) & kp.wmask;
    u[i] = (PARTY == 0) ? a : ((0u - a) & kp.wmask);  // P1: -cut(-s) mod 2^w
  }
  u[8] = 0;
  uint32_t bytes_lo = 0, bytes_hi = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t e = 0;
    if ((uint32_t)i <= kp.lx) {
      const uint32_t nxt = ((uint32_t)i < kp.lx) ? u[i + 1] : 0u;
      uint32_t vi = (u[i] + nxt - (PARTY == 0 ? 1u : 0u)) & kp.wmask;  // step 4
      uint32_t vp;                                                      // step 5 (Alg 6)
      // p > 2^w (C7), so both values already lie in [1, p): no reduction needed
      if (PARTY == 0) vp = (vi == 0) ? (1u << kp.w) : vi;
      else vp = kp.p + vi - (1u << kp.w);
      e = vp - 1u;
    }
    if (i < 4) bytes_lo |= e << (8 * i); else bytes_hi |= e << (8 * (i - 4));
  }
  const uint32_t P_lo = __byte_perm(bytes_lo, bytes_hi, tp.sel & 0xFFFFu);
  const uint32_t P_hi = __byte_perm(bytes_lo, bytes_hi, tp.sel >> 16);
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t c = byte_of(m < 4 ? P_lo : P_hi, m & 3) + 1u;
    const uint32_t rr = (PARTY == 0) ? tp.rho[m] : (kp.p - tp.rho[m]);
    W[m] = ((uint32_t)m < kp.S) ? modp_small(c * tp.r[m] + rr, kp) : 0u;  // < 257 * 257 + 257
  }
}

// P2's zero test (Alg 7 step 9): 1 iff some (W0_m + W1_m) mod p == 0.
__device__ __forceinline__ uint32_t zero_test(const uint32_t (&W0)[8], const uint32_t (&W1)[8], uint32_t p, uint32_t S) {
  uint32_t z = 0;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t s = W0[m] + W1[m];
    z |= ((uint32_t)m < S) & ((s == 0) | (s == p));
  }
  return z;
}

// Wire format: low bytes as one u64, high bits (bit 8 of W_m) as one byte.
__device__ __forceinline__ uint64_t pack_lo(const uint32_t (&W)[8]) {
  // [W0.b0, W1.b0, W0.b1, W1.b1] then merge the low halves: 3 PRMT per word
  const uint32_t lo = __byte_perm(__byte_perm(W[0], W[1], 0x5140u), __byte_perm(W[2], W[3], 0x5140u), 0x5410u);
  const uint32_t hi = __byte_perm(__byte_perm(W[4], W[5], 0x5140u), __byte_perm(W[6], W[7], 0x5140u), 0x5410u);
  return (uint64_t)lo | ((uint64_t)hi << 32);
}
__device__ __forceinline__ uint32_t pack_hi(const uint32_t (&W)[8]) {
  uint32_t h = 0;
#pragma unroll
  for (int m = 0; m < 8; ++m) h |= ((W[m] >> 8) & 1u) << m;
  return h;
}
__device__ __forceinline__ void unpack_W(uint64_t lo, uint32_t hi, uint32_t (&W)[8]) {
#pragma unroll
  for (int m = 0; m < 8; ++m) W[m] = (uint32_t)((lo >> (8 * m)) & 0xFFu) | (((hi >> m) & 1u) << 8);
}

// ---------------------------------------------------------------------------
// Vector loads / stores of 8 consecutive u64 (one group).  The caller
// guarantees 16-B alignment of the array base; full groups are 64-B aligned
// relative to it.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void load8(const uint64_t* __restrict__ p, uint64_t (&v)[8], uint32_t cnt) {
  if (cnt >= 8) {
    const ulonglong2* q = reinterpret_cast<const ulonglong2*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const ulonglong2 t = __ldg(q + i);
      v[2 * i] = t.x;
      v[2 * i + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = ((uint32_t)i < cnt) ? __ldg(p + i) : 0ull;
  }
}
__device__ __forceinline__ void store8(uint64_t* __restrict__ p, const uint64_t (&v)[8], uint32_t cnt) {
  if (cnt >= 8) {
    ulonglong2* q = reinterpret_cast<ulonglong2*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = make_ulonglong2(v[2 * i], v[2 * i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if ((uint32_t)i < cnt) p[i] = v[i];
  }
}

}  // namespace bc
