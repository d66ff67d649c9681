// bc_compact.cuh -- the compact fast path (p = 257, 8 ladder slots: guard mode at
// lx = 7, the paper's recommended key-bit width): Alg 7 steps 1-9 per element
// with SWAR byte arithmetic, table-driven shuffle and umulhi-based mod 257,
// balancing the ALU pipe (LOP3/SHF/PRMT/IADD3) against the FMA pipe (IMAD*).
//
// Per-element data flow (both computing parties; P2's zero test):
//   tape   T0..T3 (part A, 16 B) and T4, T5 (part B, 8 B): DESIGN.md "PRG tape"
//   t      = T0 >> 31                              (Alg 7 step 1)
//   Pi     = Fisher-Yates digits of T0 & 0x7fffffff, evaluated as two table
//            lookups (k7,k6,k5 | k4..k1) = (idx mod 336 | idx / 336 mod 120)
//   window = bits [f, f+15) of (-1)^t x (P0) / of -(-1)^t x (P1)     (steps 2-3)
//   bytes  c_i = u_i + u_{i+1} - 2 (P0, = v'_i - 1) or -(B_i + B_{i+1}) (P1)
//            for all 8 windows at once (steps 4-5, SWAR via a 64-bit spread multiply)
//   W_m    = ((c_{Pi(m)} + 1) r_m +- rho_m) mod 257                   (steps 6-8)
//   z      = [exists m: W0_m + W1_m in {0, 257}]                     (step 9)
#pragma once
#include "bc_device.cuh"
#include "bc_tables.cuh"

namespace bc {

constexpr int PERM_A = 336;  // 8 * 7 * 6: digits k7, k6, k5


constexpr int PERM_B = 120;  // 5 * 4 * 3 * 2: digits k4 .. k1

// Nibble selectors of the two Fisher-Yates phases (built once per CTA in smem):
// sA[0..335] / sA[336..671] = low / high halves of phase A, sB likewise (120).
__device__ __forceinline__ uint32_t fy_swap(uint32_t sel, int m, uint32_t k) {
  const uint32_t a = (sel >> (4 * m)) & 15u, b = (sel >> (4 * k)) & 15u, d = a ^ b;
  return sel ^ (d << (4 * m)) ^ (d << (4 * k));
}
__device__ __forceinline__ void build_perm_tables(uint32_t* sA, uint32_t* sB) {
  for (int i = threadIdx.x; i < PERM_A + PERM_B; i += blockDim.x) {
    uint32_t sel = 0x76543210u;
    if (i < PERM_A) {  // swaps m = 7, 6, 5 with k7 = q % 8, k6 = (q/8) % 7, k5 = q/56
      uint32_t q = (uint32_t)i;
      sel = fy_swap(sel, 7, q % 8); q /= 8;
      sel = fy_swap(sel, 6, q % 7); q /= 7;
      sel = fy_swap(sel, 5, q % 6);
      sA[i] = sel & 0xFFFFu;
      sA[PERM_A + i] = sel >> 16;
    } else {           // swaps m = 4 .. 1 with the next mixed-radix digits
      uint32_t q = (uint32_t)(i - PERM_A);
      sel = fy_swap(sel, 4, q % 5); q /= 5;
      sel = fy_swap(sel, 3, q % 4); q /= 4;
      sel = fy_swap(sel, 2, q % 3); q /= 3;
      sel = fy_swap(sel, 1, q % 2);
      sB[i - PERM_A] = sel & 0xFFFFu;
      sB[PERM_B + i - PERM_A] = sel >> 16;
    }
  }
}

// Per-element randomness in the form the slot loop consumes.
struct TapeC {
  uint32_t t;          // blinding bit
  uint32_t sel[4];     // two-phase shuffle selectors: A lo, A hi, B lo, B hi
  uint32_t rb[2];      // mask bytes r_m - 1, slot m = byte m
  uint32_t rho[8];     // reshare digits rho_m in Z_257
};

// x / 257 for any 32-bit x: floor(x * (2^40 + 1)/257 / 2^40) (exact).
__device__ __forceinline__ uint32_t div257(uint32_t x) { return __umulhi(x, 0xFF00FF01u) >> 8; }
// x / 257 for x < 2^24 with one IMAD.HI and no shift: umulhi(x, ceil(2^32 / 257)).  Since
// 2^32 - 1 = 257 * 16711935, the magic 16711936 overshoots 2^32/257 by 256/257, harmless while
// x * (256/257) / 2^32 < 1/257, i.e. x < 2^24 exactly: the first failure is x = 2^24 = 257 * 65281 - 1
// (tests/test_kernel_arith.py: exhaustive below 2^24, and that failure).
__device__ __forceinline__ uint32_t div257s(uint32_t x) { return __umulhi(x, 0xFF0100u); }

struct FbC {  // the draws a compact tape can reject, passed by value (registers, not local memory)
  uint32_t idx, w0, w1, w2;
};

template <int R>
__device__ __noinline__ FbC fallback_c(FbC d, uint64_t j, Key key) {
  FbStream<R> fb;
  fb.key = key; fb.j = j; fb.pos = 16; fb.kc = 0;
  if (d.idx >= PERM_LIMIT_8) {
    uint32_t v = fb.next() & 0x7FFFFFFFu;
    while (v >= PERM_LIMIT_8) v = fb.next() & 0x7FFFFFFFu;
    d.idx = v;
  }
  if (d.w0 >= RHO_WORD_LIMIT) { uint32_t v = fb.next(); while (v >= RHO_WORD_LIMIT) v = fb.next(); d.w0 = v; }
  if (d.w1 >= RHO_WORD_LIMIT) { uint32_t v = fb.next(); while (v >= RHO_WORD_LIMIT) v = fb.next(); d.w1 = v; }
  if (d.w2 >= RHO_WORD_LIMIT) { uint32_t v = fb.next(); while (v >= RHO_WORD_LIMIT) v = fb.next(); d.w2 = v; }
  return d;
}
// The same with the key passed by address: the table kernels take their keys as
// __grid_constant__ parameters, so &key points into the parameter bank and the eight key
// words are read inside this rare path instead of being loaded before every element's
// branch (ptxas hoisted those LDCs: ~10 issue slots per element).
template <int R>
__device__ __noinline__ FbC fallback_c(FbC d, uint64_t j, const Key* key) {
  return fallback_c<R>(d, j, *key);
}

// Compact tape (24 B): T0 = t | perm index, T1, T2 = mask bytes, reshare words
// w0 = T3 (part A), w1, w2 = T4, T5 (part B) holding rho_0..7 as base-257 digits.
template <int R>
__device__ __forceinline__ void decode_c(uint32_t T0, uint32_t T1, uint32_t T2, uint32_t w0, uint32_t w1,
                                         uint32_t w2, uint64_t j, const Key& k01, const uint32_t* sA,
                                         const uint32_t* sB, TapeC& tp) {
  tp.t = T0 >> 31;
  uint32_t idx = T0 & 0x7FFFFFFFu;
  if (__builtin_expect((idx >= PERM_LIMIT_8) | (max(w0, max(w1, w2)) >= RHO_WORD_LIMIT), 0)) {
    const FbC d = fallback_c<R>(FbC{idx, w0, w1, w2}, j, k01);
    idx = d.idx; w0 = d.w0; w1 = d.w1; w2 = d.w2;
  }
  const uint32_t hiq = idx / (uint32_t)PERM_A;               // < 2^31 / 336
  const uint32_t ia = idx - hiq * (uint32_t)PERM_A;          // (idx mod 8!) mod 336 = idx mod 336
  const uint32_t ib = hiq % (uint32_t)PERM_B;                // (idx mod 8!) / 336
  tp.sel[0] = sA[ia];
  tp.sel[1] = sA[PERM_A + ia];
  tp.sel[2] = sB[ib];
  tp.sel[3] = sB[PERM_B + ib];
  tp.rb[0] = T1;
  tp.rb[1] = T2;
  const uint32_t w[3] = {w0, w1, w2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {  // base-257 digits, least significant first
    const uint32_t q1 = div257(w[k]), q2 = div257s(q1);  // q1 < 2^24, q2 < 2^16
    tp.rho[3 * k] = w[k] - 257u * q1;
    tp.rho[3 * k + 1] = q1 - 257u * q2;
    if (k < 2) tp.rho[3 * k + 2] = q2 - 257u * div257s(q2);
  }
}

// The compact tape for the table kernels: the permutation as its index mod 8!
// (the selector is looked up in shared memory), the reshare digits as above.
template <int R>
__device__ __forceinline__ uint32_t decode_t(uint32_t T0, uint32_t w0, uint32_t w1, uint32_t w2, uint64_t j,
                                             const Key& k01, uint32_t (&rho)[8]) {
  uint32_t idx = T0 & 0x7FFFFFFFu;
  if (__builtin_expect((idx >= PERM_LIMIT_8) | (max(w0, max(w1, w2)) >= RHO_WORD_LIMIT), 0)) {
    const FbC d = fallback_c<R>(FbC{idx, w0, w1, w2}, j, k01);
    idx = d.idx; w0 = d.w0; w1 = d.w1; w2 = d.w2;
  }
  // idx mod 8! = idx - 40320 floor((idx >> 7) / 315); umulhi(x, ceil(2^32 / 315)) is exact for x < 2^24
  const uint32_t ix = idx - 40320u * __umulhi(idx >> 7, 13634817u);
  const uint32_t w[3] = {w0, w1, w2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {  // base-257 digits, least significant first
    const uint32_t q1 = div257(w[k]), q2 = div257s(q1);  // q1 < 2^24, q2 < 2^16
    rho[3 * k] = w[k] - 257u * q1;
    rho[3 * k + 1] = q1 - 257u * q2;
    if (k < 2) rho[3 * k + 2] = q2 - 257u * div257s(q2);
  }
  return ix;
}

// Windows of the party's blinded share: bits [f, f+32) of (-1)^t x (P0) or of
// -((-1)^t x) (P1) -- only bits [f, f+15) are used.
template <int PARTY>
__device__ __forceinline__ uint32_t window_of(uint64_t x, uint32_t t, uint32_t fsh, bool fhi) {
  const uint64_t nx = 0ull - x;
  const uint64_t v = (PARTY == 0) ? (t ? nx : x) : (t ? x : nx);
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  return fhi ? (hi >> fsh) : __funnelshift_r(lo, hi, fsh);
}

// Steps 3-5 for the 8 windows at once: bytes v'_i - 1 (P0) / v'_i - 1 (P1).
#ifndef BC_ADD_FMA
#define BC_ADD_FMA 2  // 0: off; 1: the mask offsets (DReLU only); 2: also the ladder sums
#endif
#ifndef BC_ADD_FMA_SEND
#define BC_ADD_FMA_SEND 0  // the same in the compact party send kernels (k_send_c)
#endif
// a + b as a multiply-add a * one + b with one = 1 read from the parameter bank (KP::one):
// ptxas cannot fold it back into an ALU-pipe IADD3, so it issues on the FMA pipe
__device__ __forceinline__ uint32_t add_fma(uint32_t a, uint32_t b, uint32_t one) { return a * one + b; }

// E = spread of a_0,a_2,a_4,a_6 into bytes 0,2,4,6 via one 64-bit multiply by
// 1 + 2^14 + 2^28 + 2^42; O likewise for a_1,a_3,a_5,a_7; 16-bit lanes then
// hold the pairwise sums without carries.  Verified exhaustively over all
// 2^15 windows (tests/test_kernel_arith.py).
template <int PARTY, bool ADDF = false>
__device__ __forceinline__ void ladder_swar(uint32_t win, uint32_t& lo, uint32_t& hi, uint32_t one = 1u) {
  constexpr uint32_t KL = 1u + (1u << 14) + (1u << 28);
  constexpr uint32_t M = 0x00FF00FFu;
  const uint32_t e = win & 0x3FFFu;
  const uint32_t o = (win >> 1) & 0x3FFFu;
  // high word of e * (KL + 2^42) for e < 2^14 is exactly (e >> 4) + (e << 10)
  const uint32_t Elo = (e * KL) & M, Ehi = ((e >> 4) + (e << 10)) & M;
  const uint32_t Olo = (o * KL) & M, Ohi = ((o >> 4) + (o << 10)) & M;
  const uint32_t Slo = __byte_perm(Elo, Ehi, 0x5432u), Shi = Ehi >> 16;  // E >> 16: a_2,a_4,a_6,0
  uint32_t ce_lo, ce_hi, co_lo, co_hi;
  if (PARTY == 0 && ADDF && BC_ADD_FMA >= 2) {  // the same sums, one add of each on the FMA pipe
    const uint32_t Oc_lo = Olo + 0x00FE00FEu, Oc_hi = Ohi + 0x00FE00FEu;
    ce_lo = Elo * one + Oc_lo; ce_hi = Ehi * one + Oc_hi;
    co_lo = Slo * one + Oc_lo; co_hi = Shi * one + Oc_hi;
  } else if (PARTY == 0) {  // u_i + u_{i+1} - 2 (mod 256) = v'_i - 1 for P0
    ce_lo = Elo + Olo + 0x00FE00FEu; ce_hi = Ehi + Ohi + 0x00FE00FEu;
    co_lo = Olo + Slo + 0x00FE00FEu; co_hi = Ohi + Shi + 0x00FE00FEu;
  } else if (ADDF && BC_ADD_FMA >= 2) {
    const uint32_t Oc_lo = 0x04000400u - Olo, Oc_hi = 0x04000400u - Ohi;
    ce_lo = Oc_lo - Elo * one; ce_hi = Oc_hi - Ehi * one;
    co_lo = Oc_lo - Slo * one; co_hi = Oc_hi - Shi * one;
  } else {           // -(B_i + B_{i+1}) (mod 256) = v'_i - 1 for P1
    ce_lo = 0x04000400u - Elo - Olo; ce_hi = 0x04000400u - Ehi - Ohi;
    co_lo = 0x04000400u - Olo - Slo; co_hi = 0x04000400u - Ohi - Shi;
  }
  // even slots from ce (bytes 0,2), odd slots from co << 8 (bytes 1,3): c ? a : b
  lo = (ce_lo & M) | ((co_lo << 8) & ~M);
  hi = (ce_hi & M) | ((co_hi << 8) & ~M);
}

// prmt.b32 straight from PTX: our selector nibbles never set the sign-replicate
// bit, so the masking __byte_perm adds is not needed.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s));
  return d;
}

// Step 6: both Fisher-Yates phases as PRMT byte gathers.  Selectors hold the
// low (output bytes 0-3) and high (bytes 4-7) nibble halves in separate words.
__device__ __forceinline__ void shuffle_bytes(uint32_t& lo, uint32_t& hi, const uint32_t (&sel)[4]) {
  const uint32_t l1 = prmt(lo, hi, sel[0]), h1 = prmt(lo, hi, sel[1]);
  lo = prmt(l1, h1, sel[2]);
  hi = prmt(l1, h1, sel[3]);
}

__device__ __forceinline__ uint32_t mod257s(uint32_t x) {  // x < 2^18
  return x - 257u * __umulhi(x, 0xFF0100u);
}

// Steps 7-8 for one party: W_m = (c_m + 1) r_m +- rho_m (mod 257), with
// r_m = rb_m + 1; the addend carries +257 / +514 so it stays positive.
template <int PARTY, bool ADDF = false>
__device__ __forceinline__ void mask_slots(uint32_t lo, uint32_t hi, const TapeC& tp, uint32_t (&W)[8], uint32_t one) {
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t c = byte_of(m < 4 ? lo : hi, m & 3);
    const uint32_t rb = byte_of(tp.rb[m >> 2], m & 3);
    const uint32_t off = (PARTY == 0) ? tp.rho[m] + 258u : 515u - tp.rho[m];
    const uint32_t add = ADDF ? add_fma(rb, off, one) : rb + off;
    W[m] = mod257s(c * (rb + 1u) + add);
  }
}

// Steps 1-9 for both computing parties and P2 on one element; returns z.
// KEEP_W: the messages are returned (transcript, both reduced to [0, 257)).
// Otherwise BC_MATERIALIZE selects how P2 tests w_m = 0:
//   0  the unreduced congruent sum -- the reshare rho cancels and the compiler
//      folds its decode away (fastest, 0.457 ms / 2^24);
//   1  (default) P0's wire value W0 in [0, 257) plus P1's congruent message:
//      rho is decoded and enters through the reduction (0.498 ms);
//   2  both wire values reduced, as the transcript path (0.514 ms).
#ifndef BC_MATERIALIZE
#define BC_MATERIALIZE 1
#endif
template <bool KEEP_W, bool ADDF = false>
__device__ __forceinline__ uint32_t elem_both(uint64_t x0, uint64_t x1, const TapeC& tp, uint32_t fsh, bool fhi, uint32_t one,
                                              uint32_t (&W0)[8], uint32_t (&W1)[8]) {
  uint32_t c_lo, c_hi, d_lo, d_hi;
  ladder_swar<0, ADDF>(window_of<0>(x0, tp.t, fsh, fhi), c_lo, c_hi, one);
  ladder_swar<1, ADDF>(window_of<1>(x1, tp.t, fsh, fhi), d_lo, d_hi, one);
  shuffle_bytes(c_lo, c_hi, tp.sel);
  shuffle_bytes(d_lo, d_hi, tp.sel);
  uint32_t vmin = 0xFFFFFFFFu;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t rb = byte_of(tp.rb[m >> 2], m & 3);
    const uint32_t r = rb + 1u;
    uint32_t a0, a1;
    if (ADDF && BC_ADD_FMA >= 1) {  // the offsets as IMADs (FMA pipe; the ALU pipe is the bound)
      a0 = add_fma(rb, tp.rho[m] + 258u, one);
      a1 = add_fma(rb, 515u - tp.rho[m], one);
    } else {
      a0 = rb + tp.rho[m] + 258u;
      a1 = rb - tp.rho[m] + 515u;
    }
    // P0's and P1's messages as integers < 2^17 congruent to W0_m, W1_m (mod 257)
    const uint32_t x0 = byte_of(m < 4 ? c_lo : c_hi, m & 3) * r + a0;   // (v'+1) r + rho + 257
    const uint32_t x1 = byte_of(m < 4 ? d_lo : d_hi, m & 3) * r + a1;   // (v'+1) r - rho + 514
    if (!KEEP_W && BC_MATERIALIZE == 1) {
      // P0's wire value W0 in [0, 257), P1's message as its congruent representative x1;
      // P2: 257 | (W0 + x1) by the multiplicative test (W0 + x1 < 2^18).  rho enters
      // through the reduction of W0, so it cannot cancel algebraically.
      vmin = min(vmin, (mod257s(x0) + x1) * 0xFF00FF01u);
    } else if (KEEP_W || BC_MATERIALIZE) {  // the wire values W in [0, 257)
      W0[m] = mod257s(x0);
      W1[m] = mod257s(x1);
      const uint32_t s = W0[m] + W1[m];
      vmin = min(vmin, s - 257u * (s >> 8));                 // 0 iff s in {0, 257}
    } else {
      // P2: w_m = W0 + W1 = 0 (mod 257)  <=>  257 | (x0 + x1)  <=>
      // (x0 + x1) * 257^-1 mod 2^32 <= floor((2^32-1)/257)   (exact for x0 + x1 < 2^19)
      vmin = min(vmin, (x0 + x1) * 0xFF00FF01u);
    }
  }
  if (!KEEP_W && BC_MATERIALIZE <= 1) return vmin <= 16711935u;
  return vmin == 0u;
}

// ---------------------------------------------------------------------------
// Table-driven variant (bc_tables.cuh; one CTA of 512 threads per SM holds the
// 210 KB of tables in shared memory).  Per element the ladder of each party is
// two shared-memory lookups instead of the SWAR arithmetic, and the shuffle is
// one lookup of the full 8! selector and one PRMT per output word.
// ---------------------------------------------------------------------------
// Window bits [f, f+32) of v (only [f, f+15) are used); FHI: f >= 32, fsh = f mod 32.
template <bool FHI>
__device__ __forceinline__ uint32_t win_at(uint64_t v, uint32_t fsh) {
  const uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
  return FHI ? (hi >> fsh) : __funnelshift_r(lo, hi, fsh);
}

// Byte offsets into the ladder sub-tables: 4 * (win mod 2^12), 4 * ((win >> 4) mod 2^11).
__device__ __forceinline__ uint32_t lad_lo_off(uint32_t win) { return (win << 2) & 0x3FFCu; }
__device__ __forceinline__ uint32_t lad_hi_off(uint32_t win) { return (win >> 2) & 0x1FFCu; }

__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t saddr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(saddr));
  return v;
}
#ifndef BC_SELH_LDS
#define BC_SELH_LDS 0  // selector high half: 1 = a second LDS.U16, 0 = a shift; measured DReLU 0.4139 -> 0.4126 ms (0), ReLU equal
#endif
#ifndef BC_SELH_LDS_SEND
#define BC_SELH_LDS_SEND 0  // the same choice in the party send kernels (elem_one_t2; measured equal)
#endif
#ifndef BC_SELH_LDS_LIT
#define BC_SELH_LDS_LIT 0  // and in the paper-literal table kernel (elem_both_tl; 0.5261 -> 0.5246 ms)
#endif
#ifndef BC_EXTRACT_DP4A
#define BC_EXTRACT_DP4A 0
#endif

// Steps 1-9 for both computing parties and P2, table form.  sbase: shared-window
// address of the tables (kPermSel at 0, kLadder after it).  ix: perm index mod 8!.
// Returns z; the messages as in elem_both.
template <bool KEEP_W, bool FHI>
__device__ __forceinline__ uint32_t elem_both_t(uint64_t x0, uint64_t x1, uint32_t t, uint32_t ix, const uint32_t (&rb)[2],
                                                const uint32_t (&rho)[8], uint32_t sbase, uint32_t fsh, uint32_t one,
                                                uint32_t (&W0)[8], uint32_t (&W1)[8]) {
  // steps 1-3: P0 windows (-1)^t x_0, P1 windows -(-1)^t x_1 (Alg 5 on -s_1, reading C3)
  const uint64_t v0 = t ? 0ull - x0 : x0;
  const uint64_t v1 = t ? x1 : 0ull - x1;
  const uint32_t wn0 = win_at<FHI>(v0, fsh), wn1 = win_at<FHI>(v1, fsh);
  constexpr uint32_t LAD = 4u * kPermN;
  // steps 3-5: ladder, pairwise sums and modulo switch as bytes v'_i - 1 (table)
  const uint32_t c_lo = lds_u32(sbase + LAD + 4u * kLadP0Lo + lad_lo_off(wn0));
  const uint32_t c_hi = lds_u32(sbase + LAD + 4u * kLadP0Hi + lad_hi_off(wn0));
  const uint32_t d_lo = lds_u32(sbase + LAD + 4u * kLadP1Lo + lad_lo_off(wn1));
  const uint32_t d_hi = lds_u32(sbase + LAD + 4u * kLadP1Hi + lad_hi_off(wn1));
  // step 6: the permutation as one selector (nibble m = source slot of slot m)
  const uint32_t sel = lds_u32(sbase + ix * 4u);
#if BC_SELH_LDS
  const uint32_t selh = lds_u16(sbase + ix * 4u + 2u);  // the high selector half as a second load (LSU, not ALU)
#else
  const uint32_t selh = sel >> 16;
#endif
  const uint32_t C_lo = prmt(c_lo, c_hi, sel), C_hi = prmt(c_lo, c_hi, selh);
  const uint32_t D_lo = prmt(d_lo, d_hi, sel), D_hi = prmt(d_lo, d_hi, selh);
  uint32_t vmin = 0xFFFFFFFFu;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
#if BC_EXTRACT_DP4A  // byte extraction as a dot product with a unit byte vector (IDP.4A, FMA pipe)
    const uint32_t unit = 1u << (8 * (m & 3));
    const uint32_t rbm = __dp4a(rb[m >> 2], unit, 0u);
    const uint32_t r = __dp4a(rb[m >> 2], unit, 1u);
    const uint32_t cm = __dp4a(m < 4 ? C_lo : C_hi, unit, 0u), dm = __dp4a(m < 4 ? D_lo : D_hi, unit, 0u);
#else
    const uint32_t rbm = byte_of(rb[m >> 2], m & 3);
    const uint32_t r = rbm + 1u;
    const uint32_t cm = byte_of(m < 4 ? C_lo : C_hi, m & 3), dm = byte_of(m < 4 ? D_lo : D_hi, m & 3);
#endif
    // steps 7-8: P0's and P1's messages as integers congruent to W0_m, W1_m (mod 257)
    const uint32_t a0 = add_fma(rbm, rho[m] + 258u, one);            // r + rho + 257
    const uint32_t a1 = add_fma(rbm, 515u - rho[m], one);            // r - rho + 514
    const uint32_t xm0 = cm * r + a0;                                 // (v'+1) r + rho + 257
    const uint32_t xm1 = dm * r + a1;                                 // (v'+1) r - rho + 514
    if (!KEEP_W && BC_MATERIALIZE == 1) {
      // P0's wire value W0 in [0, 257), P1's congruent message; P2: 257 | (W0 + x1), the sum on the FMA pipe
      vmin = min(vmin, add_fma(mod257s(xm0), xm1, one) * 0xFF00FF01u);
    } else if (KEEP_W || BC_MATERIALIZE) {
      W0[m] = mod257s(xm0);
      W1[m] = mod257s(xm1);
      vmin = min(vmin, add_fma(W0[m], W1[m], one) * 0xFF00FF01u);  // 257 | s iff s in {0, 257}
    } else {
      vmin = min(vmin, add_fma(xm0, xm1, one) * 0xFF00FF01u);
    }
  }
  return vmin <= 16711935u;  // some s_m divisible by 257: s * 257^-1 mod 2^32 <= floor((2^32-1)/257)
}

// ---- v2 of the table kernel's slot arithmetic (BC_TBL_V2) ----------------------------
// The reshare enters as congruent offsets decoded straight from the digit quotients:
//   P0: x0_m = (v'_m) r_m + o0_m, o0_m = rho_m + 257 k  (k >= 0; < 2^24)
//   P1: x1_m = (v'_m) r_m + o1_m, o1_m = 257 K - rho_m  (> 0;     <= 16710397)
// with rho_{3k} = w - 257 q1 (reduced), rho_{3k+1} = q1 - 257 q2 (== q1), rho_{3k+2}
// = q2 mod 257 (== q2), q1 = w div 257, q2 = q1 div 257.  The bytes v'-1 and r-1 are
// extracted with the +1 folded in: dp4a(word, unit byte vector, 1) = byte + 1 (IDP.4A,
// FMA pipe).  Both x0, x1 <= 65536 + 16710397 < 2^24, so div257s (exact below 2^24 only)
// reduces them; P2 tests 257 | (W0 + x1).
#ifndef BC_P2_DIST
#define BC_P2_DIST 1  // P2's test by distributivity (BC_MATERIALIZE 1): xm0 257^-1 + x1 257^-1 - q0
#endif
#ifndef BC_TBL_V2
#define BC_TBL_V2 1
#endif
template <int R>
__device__ __forceinline__ uint32_t decode_t2(uint32_t T0, uint32_t w0, uint32_t w1, uint32_t w2, uint64_t j,
                                              const Key& k01, uint32_t (&o0)[8], uint32_t (&o1)[8]) {
  uint32_t idx = T0 & 0x7FFFFFFFu;
  if (__builtin_expect((idx >= PERM_LIMIT_8) | (max(w0, max(w1, w2)) >= RHO_WORD_LIMIT), 0)) {
    const FbC d = fallback_c<R>(FbC{idx, w0, w1, w2}, j, k01);
    idx = d.idx; w0 = d.w0; w1 = d.w1; w2 = d.w2;
  }
  const uint32_t ix = idx - 40320u * __umulhi(idx >> 7, 13634817u);
  const uint32_t w[3] = {w0, w1, w2};
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const uint32_t q1 = div257(w[k]);                       // < 2^24
    o0[3 * k] = w[k] - 257u * q1;                           // rho_{3k}, reduced
    o1[3 * k] = 257u * q1 + (257u - w[k]);                  // 257 - rho_{3k} > 0
    o0[3 * k + 1] = q1;                                     // == rho_{3k+1} (mod 257)
    o1[3 * k + 1] = 16710397u - q1;                         // 257 * 65021 - q1 > 0 (q1 <= 16710396)
    if (k < 2) {
      const uint32_t q2 = div257s(q1);                      // < 2^16
      o0[3 * k + 2] = q2;                                   // == rho_{3k+2}
      o1[3 * k + 2] = 65792u - q2;                          // 257 * 256 - q2 > 0
    }
  }
  return ix;
}

#ifndef BC_BLIND_MUL
#define BC_BLIND_MUL 0  // measured: DReLU 0.4148 -> 0.4248 ms, ReLU 0.790 -> 0.797 (IMAD.WIDE is half rate)
#endif
template <bool KEEP_W, bool FHI, int MAT = BC_MATERIALIZE>
__device__ __forceinline__ uint32_t elem_both_t2(uint64_t x0, uint64_t x1, uint32_t t, uint32_t ix, const uint32_t (&rb)[2],
                                                 const uint32_t (&o0)[8], const uint32_t (&o1)[8], uint32_t sbase,
                                                 uint32_t fsh, uint32_t one, uint32_t (&W0)[8], uint32_t (&W1)[8]) {
#if BC_BLIND_MUL
  // steps 1-2 as multiplies by +-1 on the FMA pipe (IMAD.WIDE + 2 IMAD per party) instead of
  // negate-and-select on the ALU pipe: s_0 = x0 (1 - 2t), and P1's operand -s_1 = x1 (2t - 1).
  // The opaque `one` keeps ptxas from turning the products by a 0/1-derived factor into selects.
  const uint32_t m1 = 0u - one;
  const uint64_t sg = ((uint64_t)(t * m1) << 32) | (t * (m1 + m1) + one);          // 1 - 2t
  const uint64_t ng = ((uint64_t)(t * one + m1) << 32) | (t * (one + one) + m1);   // 2t - 1
  const uint64_t v0 = x0 * sg;
  const uint64_t v1 = x1 * ng;
#else
  const uint64_t v0 = t ? 0ull - x0 : x0;
  const uint64_t v1 = t ? x1 : 0ull - x1;
#endif
  const uint32_t wn0 = win_at<FHI>(v0, fsh), wn1 = win_at<FHI>(v1, fsh);
  const uint32_t four = one * 4u;  // opaque: the low offsets as IMAD (FMA pipe) + LOP3
  constexpr uint32_t LAD = 4u * kPermN;
  const uint32_t c_lo = lds_u32(sbase + LAD + 4u * kLadP0Lo + ((wn0 * four) & 0x3FFCu));
  const uint32_t c_hi = lds_u32(sbase + LAD + 4u * kLadP0Hi + lad_hi_off(wn0));
  const uint32_t d_lo = lds_u32(sbase + LAD + 4u * kLadP1Lo + ((wn1 * four) & 0x3FFCu));
  const uint32_t d_hi = lds_u32(sbase + LAD + 4u * kLadP1Hi + lad_hi_off(wn1));
  const uint32_t sel = lds_u32(sbase + ix * 4u);
#if BC_SELH_LDS
  const uint32_t selh = lds_u16(sbase + ix * 4u + 2u);
#else
  const uint32_t selh = sel >> 16;
#endif
  const uint32_t C_lo = prmt(c_lo, c_hi, sel), C_hi = prmt(c_lo, c_hi, selh);
  const uint32_t D_lo = prmt(d_lo, d_hi, sel), D_hi = prmt(d_lo, d_hi, selh);
  uint32_t vmin = 0xFFFFFFFFu;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t unit = 1u << (8 * (m & 3));
    const uint32_t r = __dp4a(rb[m >> 2], unit, 1u);                  // r_m = 1 + mask byte
    const uint32_t c1 = __dp4a(m < 4 ? C_lo : C_hi, unit, 1u);        // v'_m (P0)
    const uint32_t d1 = __dp4a(m < 4 ? D_lo : D_hi, unit, 1u);        // v'_m (P1)
    const uint32_t xm0 = c1 * r + o0[m];                              // == W0_m (mod 257)
    const uint32_t xm1 = d1 * r + o1[m];                              // == W1_m (mod 257)
    if (KEEP_W || MAT == 2) {
      W0[m] = mod257s(xm0);
      W1[m] = mod257s(xm1);
      vmin = min(vmin, add_fma(W0[m], W1[m], one) * 0xFF00FF01u);
    } else if (MAT == 1 && !BC_P2_DIST) {
      vmin = min(vmin, add_fma(mod257s(xm0), xm1, one) * 0xFF00FF01u);
    } else if (MAT == 1) {
      // P0 reduces its message: W0 = xm0 - 257 q0 with q0 = xm0 div 257 (xm0 < 2^24: div257s
      // exact).  P2 tests 257 | (W0 + x1) multiplicatively; since 257 * 257^-1 = 1 (mod 2^32),
      // (W0 + x1) 257^-1 = xm0 257^-1 + x1 257^-1 - q0 (mod 2^32): the same value, two IMADs
      // instead of forming W0 (IMAD) and the sum (IMAD) before the multiply.
      const uint32_t q0 = div257s(xm0);
      vmin = min(vmin, xm0 * 0xFF00FF01u + (xm1 * 0xFF00FF01u - q0));
    } else {
      vmin = min(vmin, add_fma(xm0, xm1, one) * 0xFF00FF01u);
    }
  }
  return vmin <= 16711935u;
}

// Alg 7 steps 1-8 for ONE computing party, table form with the V2 slot arithmetic (the
// party-separated send kernel): its message W_m in [0, 257), the wire value.  o: the party's
// reshare offsets from decode_t2 (P0 o0 = rho + 257k, P1 o1 = 257K - rho); x < 2^24.
template <int PARTY, bool FHI>
__device__ __forceinline__ void elem_one_t2(uint64_t x, uint32_t t, uint32_t ix, const uint32_t (&rb)[2],
                                            const uint32_t (&o)[8], uint32_t sbase, uint32_t fsh, uint32_t (&W)[8]) {
  const uint64_t v = PARTY == 0 ? (t ? 0ull - x : x) : (t ? x : 0ull - x);  // P1 windows -s_1 (C3)
  const uint32_t wn = win_at<FHI>(v, fsh);
  constexpr uint32_t LAD = 4u * kPermN;
  constexpr uint32_t TLO = 4u * (PARTY == 0 ? kLadP0Lo : kLadP1Lo), THI = 4u * (PARTY == 0 ? kLadP0Hi : kLadP1Hi);
  const uint32_t c_lo = lds_u32(sbase + LAD + TLO + lad_lo_off(wn));
  const uint32_t c_hi = lds_u32(sbase + LAD + THI + lad_hi_off(wn));
  const uint32_t sel = lds_u32(sbase + ix * 4u);
#if BC_SELH_LDS_SEND
  const uint32_t selh = lds_u16(sbase + ix * 4u + 2u);
#else
  const uint32_t selh = sel >> 16;
#endif
  const uint32_t C_lo = prmt(c_lo, c_hi, sel), C_hi = prmt(c_lo, c_hi, selh);
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t unit = 1u << (8 * (m & 3));
    const uint32_t r = __dp4a(rb[m >> 2], unit, 1u);            // r_m = 1 + mask byte
    const uint32_t c1 = __dp4a(m < 4 ? C_lo : C_hi, unit, 1u);  // v'_m
    W[m] = mod257s(c1 * r + o[m]);                              // steps 7-8, reduced (x < 2^24)
  }
}

// BC_TAB_TMA: the tables arrive by bulk asynchronous copies (TMA, cp.async.bulk, one elected
// thread, completion counted on an mbarrier) while every thread expands its first group's
// keystream; the first table access waits on the barrier.  Without it the CTA copies them with
// vector loads and a __syncthreads before any work.
#ifndef BC_TAB_TMA
#define BC_TAB_TMA 1
#endif
__device__ __forceinline__ void tab_bar_init(uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// issued by one thread: 4 bulk copies of the table image (each a multiple of 16 B, < 2^20 B in total)
__device__ __forceinline__ void tab_bulk_load(uint32_t* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  uint64_t g;
  asm("cvta.to.global.u64 %0, %1;" : "=l"(g) : "l"(gsrc));  // the source operand is a .global address
  const uint32_t q = ((bytes / 4u) + 15u) & ~15u;  // chunk size, 16-B multiple
  for (uint32_t off = 0; off < bytes; off += q) {
    const uint32_t sz = min(q, bytes - off);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(d + off), "l"(g + off), "r"(sz), "r"(b) : "memory");
  }
}
__device__ __forceinline__ void tab_bar_wait(uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(b) : "memory");
}


// ---- the paper-literal domain (w = lx = 7, p = 131, 8 slots, pair tape), table form ----
// Pair-tape draws of one element (T = its 8 keystream words):
// t, the permutation index mod 8!, and per slot r_m = 1 + x mod 130, rho_m = x div 130
// with x = u_m mod 17030 (u_m the 28-bit draw of slot m).  Constants of kp_literal.
template <int R>
__device__ __forceinline__ uint32_t decode_pl(const uint32_t* T, uint64_t j, const Key& k01, const KP& kp,
                                              uint32_t& t, uint32_t (&r)[8], uint32_t (&rho)[8]) {
  Draws d;
  t = T[0] >> 31;
  d.idx = T[0] & 0x7FFFFFFFu;
  uint32_t mx = 0;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const int bit = 28 * m, w = bit >> 5, sh = bit & 31;
    const uint32_t nxt = w < 6 ? T[2 + w] : 0u;
    d.um[m] = __funnelshift_r(T[1 + w], nxt, sh) & 0x0FFFFFFFu;
    d.ur[m] = 0u;
    mx = max(mx, d.um[m]);
  }
  if (__builtin_expect((d.idx >= kp.perm_lim) | (mx >= kp.pair_lim), 0)) {
    Draws f = d;
    fallback<R>(f, j, &k01, 8u, kp.perm_lim, kp.pair_lim, 1u, 0x0FFFFFFFu);
    d = f;
  }
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t x = d.um[m] - kp.pair_d * (__umulhi(d.um[m], kp.pair_mag) >> kp.pair_sh);  // u mod (p-1) p
    const uint32_t q = __umulhi(x, kp.mag_q);                                                // x div (p-1)
    r[m] = x - (kp.p - 1u) * q + 1u;
    rho[m] = q;
  }
  return d.idx - 40320u * __umulhi(d.idx >> 7, 13634817u);  // idx mod 8! (as decode_t)
}

constexpr uint32_t kInv131 = 0xC9484E2Bu;     // 131^-1 mod 2^32
constexpr uint32_t kLim131 = 32786009u;       // floor((2^32 - 1) / 131)
constexpr uint32_t kMag131 = 32786010u;       // ceil(2^32 / 131): x div 131 = umulhi(x, kMag131) for x < 2^16

// Alg 7 steps 1-9 of both computing parties and P2 in the literal domain, table form
// (bc_tables.cuh LiteralTables; sbase = its shared-window address).  P0's message
// x0_m = v'_m r_m + rho_m is reduced (W0 = x0 - 131 q0); P1's is the congruent
// x1_m = v'_m r_m + 131 - rho_m; P2 tests 131 | (W0 + x1) as the compact path does.
template <bool KEEP_W, bool FHI>
__device__ __forceinline__ uint32_t elem_both_tl(uint64_t x0, uint64_t x1, uint32_t t, uint32_t ix,
                                                 const uint32_t (&r)[8], const uint32_t (&rho)[8], uint32_t sbase,
                                                 uint32_t fsh, uint32_t (&W0)[8], uint32_t (&W1)[8]) {
  const uint64_t v0 = t ? 0ull - x0 : x0;   // steps 1-2: P0 blinds s_0
  const uint64_t v1 = t ? x1 : 0ull - x1;   // P1 windows -s_1 (Alg 5, reading C3)
  const uint32_t wn0 = win_at<FHI>(v0, fsh), wn1 = win_at<FHI>(v1, fsh);
  constexpr uint32_t LAD = 4u * kPermN;
  // steps 3-5 (table): bytes v'_i - 1; lo bytes from win bits [0, 11), hi from [4, 14)
  const uint32_t c_lo = lds_u32(sbase + LAD + 4u * kLitP0Lo + ((wn0 << 2) & 0x1FFCu));
  const uint32_t c_hi = lds_u32(sbase + LAD + 4u * kLitP0Hi + ((wn0 >> 2) & 0x0FFCu));
  const uint32_t d_lo = lds_u32(sbase + LAD + 4u * kLitP1Lo + ((wn1 << 2) & 0x1FFCu));
  const uint32_t d_hi = lds_u32(sbase + LAD + 4u * kLitP1Hi + ((wn1 >> 2) & 0x0FFCu));
  // step 6: the permutation as one selector
  const uint32_t sel = lds_u32(sbase + ix * 4u);
#if BC_SELH_LDS_LIT
  const uint32_t selh = lds_u16(sbase + ix * 4u + 2u);
#else
  const uint32_t selh = sel >> 16;
#endif
  const uint32_t C_lo = prmt(c_lo, c_hi, sel), C_hi = prmt(c_lo, c_hi, selh);
  const uint32_t D_lo = prmt(d_lo, d_hi, sel), D_hi = prmt(d_lo, d_hi, selh);
  uint32_t vmin = 0xFFFFFFFFu;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t unit = 1u << (8 * (m & 3));
    const uint32_t c1 = __dp4a(m < 4 ? C_lo : C_hi, unit, 1u);  // v'_m of P0 (byte + 1)
    const uint32_t d1 = __dp4a(m < 4 ? D_lo : D_hi, unit, 1u);  // v'_m of P1
    // steps 7-8: mask and reshare (x0 < 2^15, x1 < 2^16)
    const uint32_t xm0 = c1 * r[m] + rho[m];
    const uint32_t xm1 = d1 * r[m] + (131u - rho[m]);
    const uint32_t q0 = __umulhi(xm0, kMag131);
    if (KEEP_W) {
      W0[m] = xm0 - 131u * q0;
      W1[m] = xm1 - 131u * __umulhi(xm1, kMag131);
      vmin = min(vmin, (W0[m] + W1[m]) * kInv131);
    } else {  // step 9: (W0 + x1) 131^-1 = x0 131^-1 + x1 131^-1 - q0 (mod 2^32)
      vmin = min(vmin, xm0 * kInv131 + (xm1 * kInv131 - q0));
    }
  }
  return vmin <= kLim131;  // some W0_m + W1_m divisible by 131
}

template <int PARTY, bool ADDF = false>
__device__ __forceinline__ void elem_one(uint64_t x, const TapeC& tp, uint32_t fsh, bool fhi, uint32_t (&W)[8],
                                         uint32_t one = 1u) {
  uint32_t lo, hi;
  ladder_swar<PARTY, ADDF>(window_of<PARTY>(x, tp.t, fsh, fhi), lo, hi, one);
  shuffle_bytes(lo, hi, tp.sel);
  mask_slots<PARTY, ADDF>(lo, hi, tp, W, one);
}

}  // namespace bc
