// bc_large.cuh -- Alg 7 steps 1-9 for the large tape (lx >= 8: up to 32
// ladder slots, p < 2^33).  Full precision lx = 31, f = 0 without key bits is
// the paper's "31 * 31 ~ 1,000 bits" regime (Table 1).
//
// Per element: 7 ChaCha blocks from seed01 (large):
//   block 0     t and the Fisher-Yates draws (u16, rejection),
//   blocks 1-6  48-bit draws, 96 B per group of 8 slots: 8 masks (u -> rM = 1 +
//               u mod (p-1), rejection; the mask is r_m = rM 2^-64 mod p, i.e. rM
//               is its Montgomery form), then 8 reshares (u -> rho_m = u mod p),
// streamed 3 blocks (two slot groups) at a time through shared memory.
// Arithmetic mod p: one Montgomery product (R = 2^64) per party and slot,
// W = REDC(v' rM) = v' r; binary64 quotients for the draws.  At p = 2^32 + 15
// (the full-precision guard domain, W32) the slot runs on 32-bit operands with
// pseudo-Mersenne folds instead (fold_p15; BC_LARGE_P15).  The permutation
// is a word table per thread in shared memory ([slot][thread]) and is applied
// by evaluating slot m's source window v'_{Pi(m)} directly from the share.
#pragma once
#include <cstdint>
#include <type_traits>

#include "bc_device.cuh"

namespace bc {

constexpr uint64_t L_TAPEL = lbl("bc2.tpL2");  // seed01, 448 B / element (7 blocks at counter 7j + b)
constexpr uint64_t L_FBL = lbl("bc2.fbL2");    // seed01, large-tape fallback: u64 words, counter j*2^20 + k
constexpr uint32_t LARGE_STG_ROWS = 48;
#ifndef BC_LARGE_SLOT_UNROLL
#define BC_LARGE_SLOT_UNROLL 4  // slots per iteration of the slot loops; measured: send 9.00 -> 8.73 ms (1 -> 4)
#endif
constexpr int kLargeSlotUnroll = BC_LARGE_SLOT_UNROLL;         // keystream words staged per thread (3 blocks)
constexpr uint64_t DRAW48 = (1ull << 48) - 1ull;

struct KPL {
  uint64_t ymask;     // 2^ell - 1
  uint64_t wmask;     // 2^w - 1
  uint64_t p;         // modulus, odd, < 2^33
  uint64_t pinv;      // p^-1 mod 2^64 (Montgomery, subtractive REDC)
  uint64_t mu_p;      // floor((2^64-1) / p)      (Barrett)
  uint64_t mu_q;      // floor((2^64-1) / (p-1))
  uint64_t plim;      // floor(2^64/p) p - 1: accept u <= plim (2^64 - 1 when nothing rejects)
  uint64_t qlim;      // floor(2^64/(p-1)) (p-1) - 1
  uint64_t two_w;     // 2^w mod p (P0's image of 0, Alg 6)
  uint64_t off1;      // p - 2^w   (P1's modswitch offset, Alg 6)
  uint32_t wm32;      // 2^w - 1 as 32 bits (w <= 32)
  uint32_t f, w, S;
  double qinv_p, qoff_p;  // RN(1/p), -(2^52 + (p-1)/2)            (BC_LARGE_FPMOD)
  double qinv_q, qoff_q;  // RN(1/q'), -(2^52 + (q'-1)/2), q' = (p-1) >> s_q odd
  uint32_t s_q;           // trailing zero bits of p - 1
};

// a * b * 2^-64 mod p for a, b < p.  Subtractive REDC: m = lo p^-1 makes
// lo - lo(m p) = 0 exactly, so (ab - mp) / 2^64 = hi - hi(mp), in (-p, p).
__device__ __forceinline__ uint64_t mont(uint64_t a, uint64_t b, const KPL& kp) {
  const uint64_t lo = a * b, hi = __umul64hi(a, b);
  const uint64_t mh = __umul64hi(lo * kp.pinv, kp.p);
  return hi >= mh ? hi - mh : hi - mh + kp.p;
}

// The same product for a multiplier b shared by several a (both parties multiply by the slot's
// rM): m = (a b mod 2^64) p^-1 = a (b p^-1) mod 2^64, so with bp = b p^-1 mod 2^64 computed once
// per slot the low product a b is not needed -- the same m, the same result.
__device__ __forceinline__ uint64_t mont_shared(uint64_t a, uint64_t b, uint64_t bp, const KPL& kp) {
  const uint64_t hi = __umul64hi(a, b);
  const uint64_t mh = __umul64hi(a * bp, kp.p);
  return hi >= mh ? hi - mh : hi - mh + kp.p;
}
#ifndef BC_LARGE_MONT_SHARED
#define BC_LARGE_MONT_SHARED 1
#endif

// BC_LARGE_FPMOD = 1: the draws' reductions u mod q (u < 2^48, the tape's draws)
// by a binary64 quotient.  Write q = q' 2^s with q' odd; floor(u / q) =
// floor(v / q') with v = u >> s, and for odd q' floor(v / q') = round((v -
// (q'-1)/2) RN(1/q')): the fractions k/q' of v/q' sit at most (q'-1)/(2q') from
// the rounding point, 1/(2q') inside the tie, while the product errs by < (v/q')
// 2^-53 <= 2^-5 / q'.  So the rounded quotient is exact and so is r = u - q
// floor(u/q), with no correction step.  v - (q'-1)/2 is exact (hi word
// 0x43300000 | v_hi over v_lo is 2^52 + v), the 1.5 * 2^52 addend rounds once.
#ifndef BC_LARGE_FPMOD
#define BC_LARGE_FPMOD 1  // measured: fused full-precision DReLU 10.18 -> 9.96 ms, send 9.41 -> 9.01 ms / 2^24
#endif
__device__ __forceinline__ uint64_t fpmod48(uint64_t u, uint64_t q, uint32_t s, double qinv, double qoff) {
  const uint64_t v = u >> s;
  const double vd = __dadd_rn(__hiloint2double((int)(0x43300000u | (uint32_t)(v >> 32)), (int)(uint32_t)v), qoff);
  const double r = __fma_rn(vd, qinv, 6755399441055744.0);  // 1.5 * 2^52 + floor(v / q')
  const uint64_t qh = ((uint64_t)((uint32_t)__double2hiint(r) - 0x43380000u) << 32) | (uint32_t)__double2loint(r);
  return u - qh * q;
}

// u mod q with mu = floor((2^64-1)/q): the quotient estimate is low by at most 1.
__device__ __forceinline__ uint64_t barrett(uint64_t u, uint64_t q, uint64_t mu) {
  const uint64_t r = u - __umul64hi(u, mu) * q;
  return r >= q ? r - q : r;
}

__device__ __forceinline__ bool accept64(uint64_t u, uint64_t lim_m1) { return u <= lim_m1; }

// c-th u64 word of element j's fallback stream (rare path, kept out of line).
template <int R>
__device__ __noinline__ uint64_t fbl_word(Key k01, uint64_t j, uint32_t c) {
  uint32_t B[16];
  chacha<R>(k01, (j << 20) + (c >> 3), L_FBL, B);
  const uint32_t e = c & 7u;
  uint64_t v = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
    if ((uint32_t)i == e) v = (uint64_t)B[2 * i] | ((uint64_t)B[2 * i + 1] << 32);
  return v;
}

// Ladder source slot i of Alg 7 steps 3-5 for both parties.  s0f = s0 >> f
// and n1f = ((-s1) mod 2^ell) >> f (the blinded shares with the key-bit
// offset applied once per element), so window i is bits [i, i+w) of a 64-bit
// value with i + w <= 64 - f: one 32-bit funnel shift (i <= 31, w <= 32).
// Returns P0's c'_i and P1's d'_i in [0, p).
// W32: w = 32 (the full-precision guard domain lx = 31): every window is a whole 32-bit word,
// the masks vanish and the sums wrap mod 2^32 by themselves.
template <bool W32 = false>
__device__ __forceinline__ void slot_values(uint64_t s0f, uint64_t n1f, uint32_t i, const KPL& kp, uint64_t& c,
                                            uint64_t& d) {
  const uint32_t l0 = (uint32_t)s0f, h0 = (uint32_t)(s0f >> 32);
  const uint32_t l1 = (uint32_t)n1f, h1 = (uint32_t)(n1f >> 32);
  if (W32) {
    const bool last = i + 1 >= kp.S;                                    // slot lx has no successor
    const uint32_t a_i = __funnelshift_r(l0, h0, i);
    const uint32_t a_n = last ? 0u : __funnelshift_rc(l0, h0, i + 1);
    const uint32_t b_i = __funnelshift_r(l1, h1, i);                    // P1: -(window of -s_1), below
    const uint32_t b_n = last ? 0u : __funnelshift_rc(l1, h1, i + 1);
    const uint32_t cv = a_i + a_n - 1u;                                 // step 4 (mod 2^32)
    const uint32_t dv = 0u - (b_i + b_n);                               // -b_i - b_{i+1} (readings C3, C4)
    c = cv == 0 ? kp.two_w : (uint64_t)cv;                              // step 5 (Alg 6)
    d = (uint64_t)dv + kp.off1;
    return;
  }
  const uint32_t wm = kp.wm32;
  const uint32_t nm = i + 1 < kp.S ? wm : 0u;                          // slot lx has no successor
  const uint32_t a_i = __funnelshift_r(l0, h0, i) & wm;
  const uint32_t a_n = __funnelshift_rc(l0, h0, i + 1) & nm;
  const uint32_t b_i = (0u - (__funnelshift_r(l1, h1, i) & wm)) & wm;  // Alg 5, P1 (readings C3, C4)
  const uint32_t b_n = (0u - (__funnelshift_rc(l1, h1, i + 1) & nm)) & wm;
  const uint32_t cv = (a_i + a_n - 1u) & wm;                           // step 4: P0 carries the -1 (C8)
  const uint32_t dv = (b_i + b_n) & wm;
  c = cv == 0 ? kp.two_w : (uint64_t)cv;                               // step 5 (Alg 6), P0
  d = (uint64_t)dv + kp.off1;                                          //                 P1: p + d - 2^w
}

#ifndef BC_TPB_LARGE
#define BC_TPB_LARGE 128
#endif
constexpr int TPB_LARGE = BC_TPB_LARGE;  // threads per CTA of the large-tape kernels (shared tables are [32][TPB_LARGE])

// The per-thread permutation table.  BC_LARGE_IDX32 = 1: 32-bit entries, [slot][thread] words
// (thread t's column sits in bank t mod 32, so the Fisher-Yates swaps at random slots are
// conflict-free; round 1's byte entries in the same [slot][thread] order put four threads' columns
// in one bank word and the random-row swaps conflicted 4-way).  0: byte entries with each thread
// owning whole words ([slot / 4][thread] words, byte slot mod 4): as conflict-free, 4 KB per CTA
// instead of 16 KB.  Entry m of this thread is idx[idx_off(m)] (idx = this thread's row-0 word).
#ifndef BC_LARGE_IDX32
#define BC_LARGE_IDX32 1
#endif
#if BC_LARGE_IDX32
typedef uint32_t LargeIdx;
constexpr int kIdxWords = 32;  // table words per thread
template <int TPB_L>
__device__ __forceinline__ uint32_t idx_off(uint32_t m) { return m * (uint32_t)TPB_L; }
#else
typedef uint8_t LargeIdx;
constexpr int kIdxWords = 8;
template <int TPB_L>
__device__ __forceinline__ uint32_t idx_off(uint32_t m) { return (m >> 2) * (4u * TPB_L) + (m & 3u); }
#endif

// Per-CTA constant tables of the Fisher-Yates draws: magic[s] = ceil(2^32 / s),
// hlim[s] = floor(2^16 / s) s (the u16 rejection limit), s = 2..32.
__device__ __forceinline__ void large_tables(uint32_t* magic, uint32_t* hlim) {
  for (uint32_t s = threadIdx.x; s < 33; s += blockDim.x) {
    magic[s] = s >= 2 ? 0xFFFFFFFFu / s + 1u : 0u;
    hlim[s] = s >= 2 ? (65536u / s) * s : 0u;
  }
}

// Block 0 of element j's tape: t and step 6's Fisher-Yates permutation into
// this thread's idx column.  idx: this thread's column of a [32][TPB_L]
// LargeIdx table; stg: its column of a [32][TPB_L] word table (keystream staging, so the
// Fisher-Yates and slot loops stay rolled: the kernel must fit the instruction
// cache).  magic[s] = ceil(2^32 / s), hlim[s] = floor(2^16 / s) s.  fbc counts
// the fallback words consumed.  Returns t.
// PRE: the tape blocks through chacha_pre (pre = the (seed01, bc2.tpL2) precomputation; HI0: every
// counter 7j + b of the launch below 2^32).
template <int R, int TPB_L, bool PRE = false, bool HI0 = false>
__device__ __forceinline__ void large_block(const Key& k01, const KeyPre* pre, uint64_t ctr, uint32_t (&B)[16]) {
  if (PRE)
    chacha_pre<R, HI0>(*pre, ctr, B);
  else
    chacha<R>(k01, ctr, L_TAPEL, B);
}

template <int R, int TPB_L, bool PRE = false, bool HI0 = false>
__device__ __forceinline__ uint32_t large_perm(uint64_t j, const Key& k01, const KPL& kp, LargeIdx* idx, uint32_t* stg,
                                               const uint32_t* magic, const uint32_t* hlim, uint32_t& fbc,
                                               const KeyPre* pre = nullptr) {
  const uint32_t S = kp.S;
  uint32_t t;
  {
    uint32_t B[16];
    large_block<R, TPB_L, PRE, HI0>(k01, pre, j * 7, B);
    t = B[0] & 1u;
#pragma unroll
    for (int w = 0; w < 16; ++w) stg[w * TPB_L] = B[w];
  }
#pragma unroll 4
  for (uint32_t m = 0; m < 32; ++m) idx[idx_off<TPB_L>(m)] = (LargeIdx)m;
  // step 6: Fisher-Yates, slot m = S-1 .. 1 draws h[S-m]
#pragma unroll 1
  for (uint32_t q = 1; q < S; ++q) {
    const uint32_t m = S - q, s = m + 1;
    uint32_t d = (stg[(q >> 1) * TPB_L] >> (16 * (q & 1))) & 0xFFFFu;
    while (d >= hlim[s]) d = (uint32_t)fbl_word<R>(k01, j, fbc++) & 0xFFFFu;
    const uint32_t k = d - __umulhi(d, magic[s]) * s;
    const LargeIdx a = idx[idx_off<TPB_L>(m)], b = idx[idx_off<TPB_L>(k)];
    idx[idx_off<TPB_L>(m)] = b;
    idx[idx_off<TPB_L>(k)] = a;
  }
  return t;
}

// The same for S = 32 (lx = 31, the full-precision domains): the 31 swaps unrolled, the draws
// read from the block in registers with compile-time shifts, limits and moduli.  An element
// whose draw q rejects (~0.35 %) stages the block and finishes from q in large_perm's loop.
// BC_LARGE_PERM32: bit 0 the fused DReLU kernel, bit 1 the party send kernel, bit 2 the fused ReLU
// kernel.  Measured (2^24, with the p = 2^32 + 15 slot arithmetic): fused DReLU 7.35 -> 7.07 ms,
// fused ReLU 7.93 -> 8.07 (slower: its Beaver finish holds more registers), send 6.95 -> 6.61.
#ifndef BC_LARGE_PERM32
#define BC_LARGE_PERM32 3
#endif
template <int R, int TPB_L, bool PRE = false, bool HI0 = false>
__device__ __forceinline__ uint32_t large_perm32(uint64_t j, const Key& k01, LargeIdx* idx, uint32_t* stg,
                                                 const uint32_t* magic, const uint32_t* hlim, uint32_t& fbc,
                                                 const KeyPre* pre = nullptr) {
  uint32_t B[16];
  large_block<R, TPB_L, PRE, HI0>(k01, pre, j * 7, B);
  const uint32_t t = B[0] & 1u;
#pragma unroll
  for (uint32_t m = 0; m < 32; ++m) idx[idx_off<TPB_L>(m)] = (LargeIdx)m;
  uint32_t q0 = 32;
#pragma unroll
  for (uint32_t q = 1; q < 32; ++q) {
    const uint32_t m = 32 - q, s = m + 1;
    const uint32_t d = (B[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
    if (__builtin_expect(d >= (65536u / s) * s, 0)) {
      q0 = q;
      break;
    }
    const uint32_t k = d % s;
    const LargeIdx a = idx[idx_off<TPB_L>(m)], b = idx[idx_off<TPB_L>(k)];
    idx[idx_off<TPB_L>(m)] = b;
    idx[idx_off<TPB_L>(k)] = a;
  }
  if (__builtin_expect(q0 < 32, 0)) {  // a rejected draw: the generic loop from q0 on
#pragma unroll
    for (int w = 0; w < 16; ++w) stg[w * TPB_L] = B[w];
#pragma unroll 1
    for (uint32_t q = q0; q < 32; ++q) {
      const uint32_t m = 32 - q, s = m + 1;
      uint32_t d = (stg[(q >> 1) * TPB_L] >> (16 * (q & 1))) & 0xFFFFu;
      while (d >= hlim[s]) d = (uint32_t)fbl_word<R>(k01, j, fbc++) & 0xFFFFu;
      const uint32_t k = d - __umulhi(d, magic[s]) * s;
      const LargeIdx a = idx[idx_off<TPB_L>(m)], b = idx[idx_off<TPB_L>(k)];
      idx[idx_off<TPB_L>(m)] = b;
      idx[idx_off<TPB_L>(k)] = a;
    }
  }
  return t;
}

// 48-bit little-endian draw at byte offset `byte` (even) of the staged words.
template <int TPB_L>
__device__ __forceinline__ uint64_t draw48(const uint32_t* stg, uint32_t byte) {
  const uint32_t w = byte >> 2, sh = (byte & 3u) * 8u;  // sh is 0 or 16
  const uint32_t a = stg[w * TPB_L], b = stg[(w + 1) * TPB_L];
  return (uint64_t)__funnelshift_r(a, b, sh) | ((uint64_t)((b >> sh) & 0xFFFFu) << 32);
}

// Mask and reshare draws of slot m (its 16-slot pair of groups staged by
// large_stage): rM = Montgomery form of r_m, rho = rho_m.  Group g = m / 8 holds
// 8 mask draws then 8 reshare draws, 6 B each (96 B per group).
template <int R, int TPB_L>
__device__ __forceinline__ void large_draws(uint32_t m, uint64_t j, const Key& k01, const KPL& kp,
                                            const uint32_t* stg, uint32_t& fbc, uint64_t& rM, uint64_t& rho) {
  const uint32_t gbyte = 96u * ((m >> 3) & 1u) + 6u * (m & 7u);
  // a draw can reject only if its high 16 bits reach the limit's (probability ~2^-16):
  // one 32-bit compare on the common path, the exact test behind it
  uint64_t ur = draw48<TPB_L>(stg, gbyte);
  if (__builtin_expect((uint32_t)(ur >> 32) >= (uint32_t)(kp.qlim >> 32), 0))
    while (!accept64(ur, kp.qlim)) ur = fbl_word<R>(k01, j, fbc++) & DRAW48;
  uint64_t uq = draw48<TPB_L>(stg, gbyte + 48u);
  if (__builtin_expect((uint32_t)(uq >> 32) >= (uint32_t)(kp.plim >> 32), 0))
    while (!accept64(uq, kp.plim)) uq = fbl_word<R>(k01, j, fbc++) & DRAW48;
#if BC_LARGE_FPMOD
  rM = 1ull + fpmod48(ur, kp.p - 1ull, kp.s_q, kp.qinv_q, kp.qoff_q);  // r_m = rM 2^-64 (Montgomery form)
  rho = fpmod48(uq, kp.p, 0u, kp.qinv_p, kp.qoff_p);                    // rho_m in Z_p (p odd)
#else
  rM = 1ull + barrett(ur, kp.p - 1ull, kp.mu_q);  // r_m = rM 2^-64 (Montgomery form)
  rho = barrett(uq, kp.p, kp.mu_p);               // rho_m in Z_p
#endif
}

// The same with the slot's position inside its group of 8 a compile-time constant K (the
// group-of-8 slot loop, BC_LARGE_GROUP8): the byte offsets 6K and 48 + 6K fold into the
// staged-word index and a constant shift, G = 24 (m div 8 mod 2) is the group's first word.
// The rare exact acceptance test and redraw live out of line (large_redraw), so the common
// path is one 32-bit compare per draw.
struct Redraw {
  uint64_t u;
  uint32_t fbc;
};
template <int R>
__device__ __noinline__ Redraw large_redraw(uint64_t u, uint64_t lim_m1, Key k01, uint64_t j, uint32_t fbc) {
  while (!accept64(u, lim_m1)) u = fbl_word<R>(k01, j, fbc++) & DRAW48;
  return Redraw{u, fbc};
}
template <int TPB_L, int BYTE>
__device__ __forceinline__ uint64_t draw48c(const uint32_t* stg, uint32_t G) {
  constexpr uint32_t w = BYTE >> 2, sh = (BYTE & 3) * 8;  // sh is 0 or 16
  const uint32_t a = stg[(G + w) * TPB_L], b = stg[(G + w + 1) * TPB_L];
  if (sh == 0) return (uint64_t)a | ((uint64_t)(b & 0xFFFFu) << 32);
  return (uint64_t)__funnelshift_r(a, b, sh) | ((uint64_t)(b >> 16) << 32);
}
template <int R, int TPB_L, int K>
__device__ __forceinline__ void large_draws_k(uint32_t G, uint64_t j, const Key& k01, const KPL& kp,
                                              const uint32_t* stg, uint32_t& fbc, uint64_t& rM, uint64_t& rho) {
  uint64_t ur = draw48c<TPB_L, 6 * K>(stg, G);
  if (__builtin_expect((uint32_t)(ur >> 32) >= (uint32_t)(kp.qlim >> 32), 0)) {
    const Redraw d = large_redraw<R>(ur, kp.qlim, k01, j, fbc);
    ur = d.u;
    fbc = d.fbc;
  }
  uint64_t uq = draw48c<TPB_L, 48 + 6 * K>(stg, G);
  if (__builtin_expect((uint32_t)(uq >> 32) >= (uint32_t)(kp.plim >> 32), 0)) {
    const Redraw d = large_redraw<R>(uq, kp.plim, k01, j, fbc);
    uq = d.u;
    fbc = d.fbc;
  }
#if BC_LARGE_FPMOD
  rM = 1ull + fpmod48(ur, kp.p - 1ull, kp.s_q, kp.qinv_q, kp.qoff_q);
  rho = fpmod48(uq, kp.p, 0u, kp.qinv_p, kp.qoff_p);
#else
  rM = 1ull + barrett(ur, kp.p - 1ull, kp.mu_q);
  rho = barrett(uq, kp.p, kp.mu_p);
#endif
}
#ifndef BC_LARGE_GROUP8
#define BC_LARGE_GROUP8 1
#endif

// ---- p = 2^32 + 15: the full-precision guard domain (w = 32, W32) -------------------------
// A pseudo-Mersenne prime: 2^32 = -15 (mod p), so a 64-bit x = x1 2^32 + x0 folds to x0 - 15 x1
// with two multiply-adds and no 64 x 64 products.  The slot arithmetic below runs on 32-bit
// operands (c, d, r below 2^32: all but ~5e-9 of the slots); the rest take the generic
// Montgomery path.  Same results: every value is the same residue (tests/test_kernel_arith.py
// emulates fold_p15, mod_p15, mod_q15 and the zero test on edge and random inputs).
#ifndef BC_LARGE_P15
#define BC_LARGE_P15 1
#endif
constexpr uint64_t P15 = (1ull << 32) + 15ull;
constexpr uint32_t K15 = 0x9876543Bu;  // 2^-64 mod p: r_m = rM K15 mod p (the draw's Montgomery form, C28)

// x mod p up to one subtraction of p: y = x0 - 15 x1 lies in (-15 2^32, 2^32), as y1 2^32 + y0
// with y1 in [-15, 0]; y = y0 - 15 y1 (mod p) lies in [0, 2^32 + 225].
__device__ __forceinline__ uint64_t fold_p15(uint64_t x) {
  const uint64_t y = (uint64_t)(uint32_t)x - (x >> 32) * 15ull;  // two's complement of the signed y
  const int32_t y1 = (int32_t)(y >> 32);
  return (uint64_t)(uint32_t)y + (uint64_t)(uint32_t)(-15 * y1);
}
// u mod p and u mod (p - 1) for u < 2^48 (the tape's draws): u0 - c u1 lies in (-c 2^16, 2^32).
__device__ __forceinline__ uint64_t mod_p15(uint64_t u) {
  const int64_t v = (int64_t)(uint32_t)u - (int64_t)(15u * (uint32_t)(u >> 32));
  return (uint64_t)(v < 0 ? v + (int64_t)P15 : v);
}
__device__ __forceinline__ uint64_t mod_q15(uint64_t u) {
  const int64_t v = (int64_t)(uint32_t)u - (int64_t)(14u * (uint32_t)(u >> 32));
  return (uint64_t)(v < 0 ? v + (int64_t)(P15 - 1ull) : v);
}

// Both draws of a W32 slot on 32 bits: with m = c u1 (< 2^20), u0 - m wraps iff u0 < m and the
// residue is then (u0 - m mod 2^32) + c; rM = 1 + (ur mod (p-1)).  Returns false (take the 64-bit
// path: mod_q15 / mod_p15) when rM or rho reaches 2^32 (a sum below wraps: ~2^-28 per draw).
__device__ __forceinline__ bool draws_p15(uint64_t ur, uint64_t uq, uint32_t& rM, uint32_t& rho) {
  const uint32_t mr = 14u * (uint32_t)(ur >> 32), u0 = (uint32_t)ur;
  const uint32_t ar = u0 < mr ? 15u : 1u;  // (p - 1) - 2^32 + 1, or 1
  rM = (u0 - mr) + ar;
  const uint32_t mq = 15u * (uint32_t)(uq >> 32), v0 = (uint32_t)uq;
  const uint32_t aq = v0 < mq ? 15u : 0u;  // p - 2^32, or 0
  rho = (v0 - mq) + aq;
  return (rM >= ar) & (rho >= aq);         // no 32-bit wrap in the sums
}

// ---- p = 2^31 + 11: the paper-literal full-precision domain (w = 31, "31 * 31 ~ 1,000 bits") ----
// 2^32 = -22 (mod p) and 2^32 = -20 (mod p - 1); every operand (c, d, r, rho < p) is a 32-bit word,
// so there is no wide-operand path.  x < 2^63: y = x0 - 22 x1 in (-2^35, 2^32), y = y1 2^32 + y0 with
// y1 in [-8, 0], and y0 - 22 y1 in [0, 2^32 + 176] (< 3p): fold31 stops there, red31 finishes.
#ifndef BC_LARGE_P31
#define BC_LARGE_P31 1
#endif
constexpr uint64_t P31 = (1ull << 31) + 11ull;
constexpr uint32_t K31 = 0x5E69C906u;  // 2^-64 mod p
__device__ __forceinline__ uint64_t fold31(uint64_t x) {
  const uint64_t y = (uint64_t)(uint32_t)x - (x >> 32) * 22ull;
  const int32_t y1 = (int32_t)(y >> 32);
  return (uint64_t)(uint32_t)y + (uint64_t)(uint32_t)(-22 * y1);
}
__device__ __forceinline__ uint32_t red31(uint64_t x) {
  const uint64_t z = fold31(x);
  return (uint32_t)(z >= P31 ? (z >= 2 * P31 ? z - 2 * P31 : z - P31) : z);
}
// u mod M for u < 2^48 and M = 2^31 + c' (c = 2^32 mod M taken negative: 22 for p, 20 for p - 1):
// v = u0 - c u1 on 32 bits; a wrap adds M - 2^32 + ... = c back after subtracting M once.
template <uint32_t M, uint32_t C>
__device__ __forceinline__ uint32_t mod31(uint64_t u) {
  const uint32_t m = C * (uint32_t)(u >> 32), u0 = (uint32_t)u;
  const uint32_t v = u0 - m;
  return v - (v >= M ? M : 0u) + (u0 < m ? C : 0u);
}

// The exact acceptance tests and redraws of a slot's two 48-bit draws, out of line, in draw order
// (r_m's, then rho_m's: the fallback stream's order); the W32 slot calls it when a draw's high
// 16 bits reach the limit's (the only way it can reject).
struct Redraw2 {
  uint64_t ur, uq;
  uint32_t fbc;
};
template <int R>
__device__ __noinline__ Redraw2 large_redraw2(uint64_t ur, uint64_t uq, uint64_t qlim, uint64_t plim, Key k01,
                                              uint64_t j, uint32_t fbc) {
  while (!accept64(ur, qlim)) ur = fbl_word<R>(k01, j, fbc++) & DRAW48;
  while (!accept64(uq, plim)) uq = fbl_word<R>(k01, j, fbc++) & DRAW48;
  return Redraw2{ur, uq, fbc};
}
// Blocks 1 + 3h .. 3 + 3h (slot groups 2h, 2h + 1) into staged rows 0..47.
template <int R, int TPB_L, bool PRE = false, bool HI0 = false>
__device__ __forceinline__ void large_stage(uint32_t h, uint64_t j, const Key& k01, uint32_t* stg,
                                            const KeyPre* pre = nullptr) {
#pragma unroll 1
  for (uint32_t b = 0; b < 3; ++b) {
    uint32_t B[16];
    large_block<R, TPB_L, PRE, HI0>(k01, pre, j * 7 + 1 + 3 * h + b, B);
#pragma unroll
    for (int w = 0; w < 16; ++w) stg[(16 * b + w) * TPB_L] = B[w];
  }
}

// Alg 7 steps 1-9 for element j with shares x0, x1 (both computing parties and
// P2's zero test): returns DReLU' (bit 0) and t (bit 1).
template <int R, bool TRANSCRIPT, int TPB_L, bool PRE = false, bool HI0 = false, bool W32 = false, bool RELU = false,
          bool L31 = false>
__device__ __forceinline__ uint32_t elem_large(uint64_t x0, uint64_t x1, uint64_t j, const Key& k01, const KPL& kp,
                                               LargeIdx* idx, uint32_t* stg, const uint32_t* magic,
                                               const uint32_t* hlim, uint64_t* w0, uint64_t* w1,
                                               const KeyPre* pre = nullptr) {
  const uint32_t S = kp.S;
  uint32_t fbc = 0;  // fallback words consumed
  const uint32_t t = (W32 || L31) && (BC_LARGE_PERM32 & (RELU ? 4 : 1)) ? large_perm32<R, TPB_L, PRE, HI0>(j, k01, idx, stg, magic, hlim, fbc, pre)
                                                   : large_perm<R, TPB_L, PRE, HI0>(j, k01, kp, idx, stg, magic, hlim, fbc, pre);
  // steps 1-2: blind both shares by (-1)^t
  const uint64_t s0 = t ? (0ull - x0) & kp.ymask : x0 & kp.ymask;
  const uint64_t s1 = t ? (0ull - x1) & kp.ymask : x1 & kp.ymask;
  const uint64_t s0f = s0 >> kp.f, n1f = ((0ull - s1) & kp.ymask) >> kp.f;
  uint32_t z = 0;
  // steps 6-9 for slot m with its draws rM, rho
  auto slot = [&](uint32_t m, uint64_t rM, uint64_t rho) {
      uint64_t c, d;
      slot_values<W32>(s0f, n1f, idx[idx_off<TPB_L>(m)], kp, c, d);           // v'_{Pi(m)} of each party
      const uint64_t rp = rM * kp.pinv;                              // shared by both products
      uint64_t W0 = (BC_LARGE_MONT_SHARED ? mont_shared(c, rM, rp, kp) : mont(c, rM, kp)) + rho;  // steps 7-8, P0
      W0 = W0 >= kp.p ? W0 - kp.p : W0;
      uint64_t W1 = (BC_LARGE_MONT_SHARED ? mont_shared(d, rM, rp, kp) : mont(d, rM, kp)) + (kp.p - rho);  // P1
      if (TRANSCRIPT) {
        W1 = W1 >= kp.p ? W1 - kp.p : W1;
        w0[m] = W0;
        w1[m] = W1;
        const uint64_t sum = W0 + W1;                                // step 9 (P2): w_m = 0 mod p?
        z |= (sum == 0 || sum == kp.p) ? 1u : 0u;
      } else {
        const uint64_t sum = W0 + W1;  // P0's W0 in [0, p) + P1's congruent x1 in (0, 2p]: 0 mod p iff p or 2p
        z |= (sum == kp.p || sum == 2 * kp.p) ? 1u : 0u;
      }
  };
  if (L31 && !TRANSCRIPT && BC_LARGE_P31) {
    // p = 2^31 + 11, S = 32: r = rM K31, P0's wire value W0 = c r + rho in [0, p), P1's message
    // d r + (p - rho) folded (below 2^32 + 177); P2: s = W0 + W1 < 2^33 is 0 mod p iff
    // s0 - 22 s1 (in [-22, 2^32)) is 0 or p.
    auto slot31 = [&](auto Kc, uint32_t G, uint32_t m) {
      constexpr int K = decltype(Kc)::value;
      uint64_t ur = draw48c<TPB_L, 6 * K>(stg, G), uq = draw48c<TPB_L, 48 + 6 * K>(stg, G);
      if (__builtin_expect(((uint32_t)(ur >> 32) >= (uint32_t)(kp.qlim >> 32)) |
                           ((uint32_t)(uq >> 32) >= (uint32_t)(kp.plim >> 32)), 0)) {
        const Redraw2 dr = large_redraw2<R>(ur, uq, kp.qlim, kp.plim, k01, j, fbc);
        ur = dr.ur;
        uq = dr.uq;
        fbc = dr.fbc;
      }
      const uint32_t rM = 1u + mod31<(uint32_t)(P31 - 1), 20u>(ur);    // Montgomery form of r_m (C28)
      const uint32_t rho = mod31<(uint32_t)P31, 22u>(uq);
      uint64_t c, d;
      slot_values<false>(s0f, n1f, idx[idx_off<TPB_L>(m)], kp, c, d);         // c in [1, 2^31], d in [11, p)
      const uint32_t r = red31((uint64_t)rM * K31);
      const uint32_t W0 = red31((uint64_t)(uint32_t)c * r + rho);      // P0's wire value
      const uint64_t W1 = fold31((uint64_t)(uint32_t)d * r + (P31 - rho));
      const uint64_t sm = W0 + W1;
      const int64_t tz = (int64_t)(uint32_t)sm - 22ll * (int64_t)(sm >> 32);
      z |= (tz == 0 || tz == (int64_t)P31) ? 1u : 0u;
    };
#pragma unroll 1
    for (uint32_t h = 0; h < 2; ++h) {
      large_stage<R, TPB_L, PRE, HI0>(h, j, k01, stg, pre);
#pragma unroll 1
      for (uint32_t g8 = 16 * h; g8 < 16 * h + 16; g8 += 8) {
        const uint32_t G = 24u * ((g8 >> 3) & 1u);
        using std::integral_constant;
        slot31(integral_constant<int, 0>{}, G, g8 + 0); slot31(integral_constant<int, 1>{}, G, g8 + 1);
        slot31(integral_constant<int, 2>{}, G, g8 + 2); slot31(integral_constant<int, 3>{}, G, g8 + 3);
        slot31(integral_constant<int, 4>{}, G, g8 + 4); slot31(integral_constant<int, 5>{}, G, g8 + 5);
        slot31(integral_constant<int, 6>{}, G, g8 + 6); slot31(integral_constant<int, 7>{}, G, g8 + 7);
      }
    }
    return z | (t << 1);
  }
  if (W32 && !TRANSCRIPT && BC_LARGE_P15) {
    // p = 2^32 + 15, S = 32 (every slot group full).  Per slot: r = rM K15, P0's wire value
    // W0 = c r + rho in [0, p), P1's message d r + (p - rho) folded (congruent, below
    // 2^32 + 226); P2: s = W0 + W1 < 3 2^32 is 0 mod p iff s0 - 15 s1 = 0 (|s0 - 15 s1| < p).
    const uint32_t l0 = (uint32_t)s0f, h0 = (uint32_t)(s0f >> 32), l1 = (uint32_t)n1f, h1 = (uint32_t)(n1f >> 32);
    // Slot g8 + K of the staged groups: one branch per slot covers the draws' rejection (the
    // exact test and the fallback stream, in draw order) and every operand at or above 2^32.
    auto slot15 = [&](auto Kc, uint32_t G, uint32_t m) {
      constexpr int K = decltype(Kc)::value;
      uint64_t ur = draw48c<TPB_L, 6 * K>(stg, G), uq = draw48c<TPB_L, 48 + 6 * K>(stg, G);
      const bool rej = ((uint32_t)(ur >> 32) >= (uint32_t)(kp.qlim >> 32)) | ((uint32_t)(uq >> 32) >= (uint32_t)(kp.plim >> 32));
      uint32_t rM32, rho32;                                            // Montgomery form of r_m (C28), rho_m
      const bool ok = draws_p15(ur, uq, rM32, rho32);
      // steps 3-5 for slot i = Pi(m) (slot_values<true> on 32 bits): c = 2^32 and d >= 2^32 are flagged
      const uint32_t i = idx[idx_off<TPB_L>(m)];
      const bool last = i == 31u;                                      // slot lx has no successor
      const uint32_t cv = __funnelshift_r(l0, h0, i) + (last ? 0u : __funnelshift_rc(l0, h0, i + 1)) - 1u;
      const uint32_t d32 = 15u - (__funnelshift_r(l1, h1, i) + (last ? 0u : __funnelshift_rc(l1, h1, i + 1)));
      const uint64_t rz = fold_p15((uint64_t)rM32 * K15);              // = r_m when below 2^32
      const uint32_t r = (uint32_t)rz;
      uint64_t W0 = fold_p15((uint64_t)cv * r + rho32);                // c r + rho < 2^64
      W0 = W0 >= P15 ? W0 - P15 : W0;                                  // P0's wire value
      const uint64_t W1 = fold_p15((uint64_t)d32 * r + (P15 - rho32));
      const uint64_t sm = W0 + W1;
      uint32_t zm = (uint32_t)sm == 15u * (uint32_t)(sm >> 32) ? 1u : 0u;
      if (__builtin_expect(rej | !ok | (cv == 0u) | (d32 < 15u) | ((uint32_t)(rz >> 32) != 0u), 0)) {
        if (rej) {
          const Redraw2 dr = large_redraw2<R>(ur, uq, kp.qlim, kp.plim, k01, j, fbc);
          ur = dr.ur;
          uq = dr.uq;
          fbc = dr.fbc;
        }
        uint64_t c, d;
        slot_values<true>(s0f, n1f, i, kp, c, d);
        const uint64_t rM = 1ull + mod_q15(ur), rho = mod_p15(uq);
        const uint64_t rp = rM * kp.pinv;
        uint64_t V0 = mont_shared(c, rM, rp, kp) + rho;
        V0 = V0 >= kp.p ? V0 - kp.p : V0;
        const uint64_t V1 = mont_shared(d, rM, rp, kp) + (kp.p - rho);
        const uint64_t sum = V0 + V1;
        zm = (sum == kp.p || sum == 2 * kp.p) ? 1u : 0u;
      }
      z |= zm;
    };
#pragma unroll 1
    for (uint32_t h = 0; h < 2; ++h) {
      large_stage<R, TPB_L, PRE, HI0>(h, j, k01, stg, pre);
#pragma unroll 1
      for (uint32_t g8 = 16 * h; g8 < 16 * h + 16; g8 += 8) {
        const uint32_t G = 24u * ((g8 >> 3) & 1u);
        using std::integral_constant;
        slot15(integral_constant<int, 0>{}, G, g8 + 0); slot15(integral_constant<int, 1>{}, G, g8 + 1);
        slot15(integral_constant<int, 2>{}, G, g8 + 2); slot15(integral_constant<int, 3>{}, G, g8 + 3);
        slot15(integral_constant<int, 4>{}, G, g8 + 4); slot15(integral_constant<int, 5>{}, G, g8 + 5);
        slot15(integral_constant<int, 6>{}, G, g8 + 6); slot15(integral_constant<int, 7>{}, G, g8 + 7);
      }
    }
    return z | (t << 1);
  }
  if (BC_LARGE_GROUP8) {
#pragma unroll 1
    for (uint32_t h = 0; 16 * h < S; ++h) {
      large_stage<R, TPB_L, PRE, HI0>(h, j, k01, stg, pre);
      const uint32_t mend = min(S, 16 * h + 16);
#pragma unroll 1
      for (uint32_t g8 = 16 * h; g8 < mend; g8 += 8) {
        const uint32_t G = 24u * ((g8 >> 3) & 1u);
        uint64_t rM, rho;
#define BC_LARGE_SLOT(K)                                                     \
        if (g8 + K < mend) {                                                 \
          large_draws_k<R, TPB_L, K>(G, j, k01, kp, stg, fbc, rM, rho);      \
          slot(g8 + K, rM, rho);                                             \
        }
        BC_LARGE_SLOT(0) BC_LARGE_SLOT(1) BC_LARGE_SLOT(2) BC_LARGE_SLOT(3)
        BC_LARGE_SLOT(4) BC_LARGE_SLOT(5) BC_LARGE_SLOT(6) BC_LARGE_SLOT(7)
#undef BC_LARGE_SLOT
      }
    }
    return z | (t << 1);
  }
#pragma unroll 1
  for (uint32_t h = 0; 16 * h < S; ++h) {
    large_stage<R, TPB_L, PRE, HI0>(h, j, k01, stg, pre);
    const uint32_t mend = min(S, 16 * h + 16);
#pragma unroll kLargeSlotUnroll
    for (uint32_t m = 16 * h; m < mend; ++m) {
      uint64_t rM, rho;
      large_draws<R, TPB_L>(m, j, k01, kp, stg, fbc, rM, rho);
      uint64_t c, d;
      slot_values<W32>(s0f, n1f, idx[idx_off<TPB_L>(m)], kp, c, d);           // v'_{Pi(m)} of each party
      const uint64_t rp = rM * kp.pinv;                              // shared by both products
      uint64_t W0 = (BC_LARGE_MONT_SHARED ? mont_shared(c, rM, rp, kp) : mont(c, rM, kp)) + rho;  // steps 7-8, P0
      W0 = W0 >= kp.p ? W0 - kp.p : W0;
      uint64_t W1 = (BC_LARGE_MONT_SHARED ? mont_shared(d, rM, rp, kp) : mont(d, rM, kp)) + (kp.p - rho);  // P1
      if (TRANSCRIPT) {
        W1 = W1 >= kp.p ? W1 - kp.p : W1;
        w0[m] = W0;
        w1[m] = W1;
        const uint64_t sum = W0 + W1;                                // step 9 (P2): w_m = 0 mod p?
        z |= (sum == 0 || sum == kp.p) ? 1u : 0u;
      } else {
        // P0's wire value W0 in [0, p) and P1's message as its congruent representative
        // in (0, 2p] (as the compact path, BC_MATERIALIZE=1): W0 + W1 in (0, 3p), and
        // w_m = 0 mod p iff the sum is p or 2p.  rho enters through W0's reduction.
        const uint64_t sum = W0 + W1;
        z |= (sum == kp.p || sum == 2 * kp.p) ? 1u : 0u;
      }
    }
  }
  return z | (t << 1);
}

// Alg 7 steps 1-8 for ONE computing party (the party-separated send phase):
// the message W_m, m < S, as 32-bit low words lo[m * stride] (slot-major wire
// planes) and bit m of the returned high-bit word (bit 32 of W_m; p < 2^33).
// Returns t in bit 32 of the result.
template <int R, int PARTY, int TPB_L, bool W32 = false, bool PRE = false, bool HI0 = false, bool L31 = false>
__device__ __forceinline__ uint64_t elem_large_party(uint64_t x, uint64_t j, const Key& k01, const KPL& kp,
                                                     LargeIdx* idx, uint32_t* stg, const uint32_t* magic,
                                                     const uint32_t* hlim, uint32_t* lo, uint64_t stride,
                                                     const KeyPre* pre = nullptr) {
  const uint32_t S = kp.S;
  uint32_t fbc = 0;
  const uint32_t t = (W32 || L31) && (BC_LARGE_PERM32 & 2) ? large_perm32<R, TPB_L, PRE, HI0>(j, k01, idx, stg, magic, hlim, fbc, pre)
                                                   : large_perm<R, TPB_L, PRE, HI0>(j, k01, kp, idx, stg, magic, hlim, fbc, pre);
  const uint64_t s = t ? (0ull - x) & kp.ymask : x & kp.ymask;                  // steps 1-2
  // P0 reads windows of s, P1 of (-s) mod 2^ell (Alg 5, readings C3, C4)
  const uint64_t sf = (PARTY == 0 ? s : (0ull - s) & kp.ymask) >> kp.f;
  uint32_t hib = 0;
  if (L31 && BC_LARGE_P31) {  // p = 2^31 + 11, S = 32: the slot arithmetic of elem_large's L31 path
    auto slot31 = [&](auto Kc, uint32_t G, uint32_t m) {
      constexpr int K = decltype(Kc)::value;
      uint64_t ur = draw48c<TPB_L, 6 * K>(stg, G), uq = draw48c<TPB_L, 48 + 6 * K>(stg, G);
      if (__builtin_expect(((uint32_t)(ur >> 32) >= (uint32_t)(kp.qlim >> 32)) |
                           ((uint32_t)(uq >> 32) >= (uint32_t)(kp.plim >> 32)), 0)) {
        const Redraw2 dr = large_redraw2<R>(ur, uq, kp.qlim, kp.plim, k01, j, fbc);
        ur = dr.ur;
        uq = dr.uq;
        fbc = dr.fbc;
      }
      const uint32_t rM = 1u + mod31<(uint32_t)(P31 - 1), 20u>(ur);
      const uint32_t rho = mod31<(uint32_t)P31, 22u>(uq);
      uint64_t c, d;
      slot_values<false>(sf, sf, idx[idx_off<TPB_L>(m)], kp, c, d);           // one of the two is this party's
      const uint32_t r = red31((uint64_t)rM * K31);
      const uint32_t W = red31((uint64_t)(uint32_t)(PARTY == 0 ? c : d) * r + (PARTY == 0 ? (uint64_t)rho : P31 - rho));
      lo[m * stride] = W;                                               // p < 2^32: no bit-32 plane
    };
#pragma unroll 1
    for (uint32_t h = 0; h < 2; ++h) {
      large_stage<R, TPB_L, PRE, HI0>(h, j, k01, stg, pre);
#pragma unroll 1
      for (uint32_t g8 = 16 * h; g8 < 16 * h + 16; g8 += 8) {
        const uint32_t G = 24u * ((g8 >> 3) & 1u);
        using std::integral_constant;
        slot31(integral_constant<int, 0>{}, G, g8 + 0); slot31(integral_constant<int, 1>{}, G, g8 + 1);
        slot31(integral_constant<int, 2>{}, G, g8 + 2); slot31(integral_constant<int, 3>{}, G, g8 + 3);
        slot31(integral_constant<int, 4>{}, G, g8 + 4); slot31(integral_constant<int, 5>{}, G, g8 + 5);
        slot31(integral_constant<int, 6>{}, G, g8 + 6); slot31(integral_constant<int, 7>{}, G, g8 + 7);
      }
    }
    return (uint64_t)hib | ((uint64_t)t << 32);
  }
  if (W32 && BC_LARGE_P15) {  // p = 2^32 + 15, S = 32: the pseudo-Mersenne slot arithmetic of elem_large
    const uint32_t l0 = (uint32_t)sf, h0 = (uint32_t)(sf >> 32);
    auto slot15 = [&](auto Kc, uint32_t G, uint32_t m) {
      constexpr int K = decltype(Kc)::value;
      uint64_t ur = draw48c<TPB_L, 6 * K>(stg, G), uq = draw48c<TPB_L, 48 + 6 * K>(stg, G);
      const bool rej = ((uint32_t)(ur >> 32) >= (uint32_t)(kp.qlim >> 32)) | ((uint32_t)(uq >> 32) >= (uint32_t)(kp.plim >> 32));
      uint32_t rM32, rho32;
      const bool ok = draws_p15(ur, uq, rM32, rho32);
      const uint32_t i = idx[idx_off<TPB_L>(m)];
      const uint32_t ws = __funnelshift_r(l0, h0, i) + (i == 31u ? 0u : __funnelshift_rc(l0, h0, i + 1));
      const uint32_t v32 = PARTY == 0 ? ws - 1u : 15u - ws;            // c (flag c = 2^32) / d (flag d >= 2^32)
      const bool vbad = PARTY == 0 ? v32 == 0u : v32 < 15u;
      const uint64_t rz = fold_p15((uint64_t)rM32 * K15);              // r_m when below 2^32
      uint64_t W = fold_p15((uint64_t)v32 * (uint32_t)rz + (PARTY == 0 ? (uint64_t)rho32 : P15 - rho32));
      W = W >= P15 ? W - P15 : W;                                      // steps 7-8, wire value in [0, p)
      if (__builtin_expect(rej | !ok | vbad | ((uint32_t)(rz >> 32) != 0u), 0)) {
        if (rej) {
          const Redraw2 dr = large_redraw2<R>(ur, uq, kp.qlim, kp.plim, k01, j, fbc);
          ur = dr.ur;
          uq = dr.uq;
          fbc = dr.fbc;
        }
        uint64_t c, d;
        slot_values<true>(sf, sf, i, kp, c, d);
        const uint64_t rM = 1ull + mod_q15(ur), rho = mod_p15(uq);
        W = mont(PARTY == 0 ? c : d, rM, kp) + (PARTY == 0 ? rho : kp.p - rho);  // generic path
        W = W >= kp.p ? W - kp.p : W;
      }
      lo[m * stride] = (uint32_t)W;
      hib |= (uint32_t)(W >> 32) << m;
    };
#pragma unroll 1
    for (uint32_t h = 0; h < 2; ++h) {
      large_stage<R, TPB_L, PRE, HI0>(h, j, k01, stg, pre);
#pragma unroll 1
      for (uint32_t g8 = 16 * h; g8 < 16 * h + 16; g8 += 8) {
        const uint32_t G = 24u * ((g8 >> 3) & 1u);
        using std::integral_constant;
        slot15(integral_constant<int, 0>{}, G, g8 + 0); slot15(integral_constant<int, 1>{}, G, g8 + 1);
        slot15(integral_constant<int, 2>{}, G, g8 + 2); slot15(integral_constant<int, 3>{}, G, g8 + 3);
        slot15(integral_constant<int, 4>{}, G, g8 + 4); slot15(integral_constant<int, 5>{}, G, g8 + 5);
        slot15(integral_constant<int, 6>{}, G, g8 + 6); slot15(integral_constant<int, 7>{}, G, g8 + 7);
      }
    }
    return (uint64_t)hib | ((uint64_t)t << 32);
  }
  auto slot = [&](uint32_t m, uint64_t rM, uint64_t rho) {
      uint64_t c, d;
      slot_values<W32>(sf, sf, idx[idx_off<TPB_L>(m)], kp, c, d);             // one of the two is this party's
      uint64_t W = PARTY == 0 ? mont(c, rM, kp) + rho : mont(d, rM, kp) + (kp.p - rho);  // steps 7-8
      W = W >= kp.p ? W - kp.p : W;
      lo[m * stride] = (uint32_t)W;
      hib |= (uint32_t)(W >> 32) << m;
  };
  if (BC_LARGE_GROUP8) {
#pragma unroll 1
    for (uint32_t h = 0; 16 * h < S; ++h) {
      large_stage<R, TPB_L, PRE, HI0>(h, j, k01, stg, pre);
      const uint32_t mend = min(S, 16 * h + 16);
#pragma unroll 1
      for (uint32_t g8 = 16 * h; g8 < mend; g8 += 8) {
        const uint32_t G = 24u * ((g8 >> 3) & 1u);
        uint64_t rM, rho;
#define BC_LARGE_SLOT(K)                                                     \
        if (g8 + K < mend) {                                                 \
          large_draws_k<R, TPB_L, K>(G, j, k01, kp, stg, fbc, rM, rho);      \
          slot(g8 + K, rM, rho);                                             \
        }
        BC_LARGE_SLOT(0) BC_LARGE_SLOT(1) BC_LARGE_SLOT(2) BC_LARGE_SLOT(3)
        BC_LARGE_SLOT(4) BC_LARGE_SLOT(5) BC_LARGE_SLOT(6) BC_LARGE_SLOT(7)
#undef BC_LARGE_SLOT
      }
    }
    return (uint64_t)hib | ((uint64_t)t << 32);
  }
#pragma unroll 1
  for (uint32_t h = 0; 16 * h < S; ++h) {
    large_stage<R, TPB_L, PRE, HI0>(h, j, k01, stg, pre);
    const uint32_t mend = min(S, 16 * h + 16);
#pragma unroll kLargeSlotUnroll
    for (uint32_t m = 16 * h; m < mend; ++m) {
      uint64_t rM, rho;
      large_draws<R, TPB_L>(m, j, k01, kp, stg, fbc, rM, rho);
      uint64_t c, d;
      slot_values<W32>(sf, sf, idx[idx_off<TPB_L>(m)], kp, c, d);             // one of the two is this party's
      uint64_t W = PARTY == 0 ? mont(c, rM, kp) + rho : mont(d, rM, kp) + (kp.p - rho);  // steps 7-8
      W = W >= kp.p ? W - kp.p : W;
      lo[m * stride] = (uint32_t)W;
      hib |= (uint32_t)(W >> 32) << m;
    }
  }
  return (uint64_t)hib | ((uint64_t)t << 32);
}

}  // namespace bc
