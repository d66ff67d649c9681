// bc_compact.cuh -- the compact fast path (p = 257, 8 ladder slots: guard mode at
// lx = 7, the paper's recommended key-bit width): Alg 7 steps 1-9 per element
// with SWAR byte arithmetic, table-driven shuffle and umulhi-based mod 257,
// balancing the ALU pipe (LOP3/SHF/PRMT/IADD3) against the FMA pipe (IMAD*).
//
// Per-element data flow (both computing parties; P2's zero test):
//   tape   T0..T6 (7 of the element's 8 keystream words)
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

namespace bc {

constexpr int PERM_A = 336;  // 8 * 7 * 6: digits k7, k6, k5
constexpr int PERM_B = 120;  // 5 * 4 * 3 * 2: digits k4 .. k1

// Nibble selectors of the two Fisher-Yates phases (built once per CTA in smem).
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
      sA[i] = sel;
    } else {           // swaps m = 4 .. 1 with the next mixed-radix digits
      uint32_t q = (uint32_t)(i - PERM_A);
      sel = fy_swap(sel, 4, q % 5); q /= 5;
      sel = fy_swap(sel, 3, q % 4); q /= 4;
      sel = fy_swap(sel, 2, q % 3); q /= 3;
      sel = fy_swap(sel, 1, q % 2);
      sB[i - PERM_A] = sel;
    }
  }
}

// Per-element randomness in the form the slot loop consumes.
struct TapeC {
  uint32_t t;          // blinding bit
  uint32_t selA, selB; // two-phase shuffle selectors (nibbles)
  uint32_t r[4];       // 16-bit lanes: slot 2j -> lane 0 of r[j], slot 2j+1 -> lane 1
  uint32_t a0[4];      // lanes of r_m + rho_m + 257      (P0 addend)
  uint32_t a1[4];      // lanes of r_m - rho_m + 514      (P1 addend)
};

// Halfword == 0xFFFF detector (exact as a boolean): haszero16(~w).
__device__ __forceinline__ uint32_t has_ffff(uint32_t w) { return (0u - w - 0x00010002u) & w & 0x80008000u; }

template <int R>
__device__ __forceinline__ void decode_c(uint32_t T0, uint32_t T1, uint32_t T2, uint32_t w3, uint32_t w4,
                                         uint32_t w5, uint32_t w6, uint64_t j, const Key& k01,
                                         const uint32_t* sA, const uint32_t* sB, TapeC& tp) {
  tp.t = T0 >> 31;
  uint32_t idx = T0 & 0x7FFFFFFFu;
  const uint32_t hz = has_ffff(w3) | has_ffff(w4) | has_ffff(w5) | has_ffff(w6);
  if (__builtin_expect((hz != 0) | (idx >= PERM_LIMIT_8), 0)) {
    Draws d;
    d.idx = idx;
    d.ur[0] = w3 & 0xFFFFu; d.ur[1] = w3 >> 16; d.ur[2] = w4 & 0xFFFFu; d.ur[3] = w4 >> 16;
    d.ur[4] = w5 & 0xFFFFu; d.ur[5] = w5 >> 16; d.ur[6] = w6 & 0xFFFFu; d.ur[7] = w6 >> 16;
    fallback<R>(d, j, k01, 8, PERM_LIMIT_8, 0, 65535u);
    idx = d.idx;
    w3 = d.ur[0] | (d.ur[1] << 16); w4 = d.ur[2] | (d.ur[3] << 16);
    w5 = d.ur[4] | (d.ur[5] << 16); w6 = d.ur[6] | (d.ur[7] << 16);
  }
  const uint32_t hiq = idx / (uint32_t)PERM_A;               // < 2^31 / 336
  tp.selA = sA[idx - hiq * (uint32_t)PERM_A];                // (idx mod 8!) mod 336 = idx mod 336
  tp.selB = sB[hiq % (uint32_t)PERM_B];                      // (idx mod 8!) / 336
  const uint32_t U[4] = {w3, w4, w5, w6};
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    // r_m - 1 bytes of T1 (slots 0..3) / T2 (slots 4..7) spread into 16-bit lanes
    const uint32_t rb = __byte_perm(jj < 2 ? T1 : T2, 0u, (jj & 1) ? 0x4342u : 0x4140u);
    const uint32_t L = U[jj] & 0x00FF00FFu;                  // low bytes l of the u16 draws
    const uint32_t H = __byte_perm(U[jj], 0u, 0x4341u);      // high bytes h; rho = u mod 257 = l - h mod 257
    tp.r[jj] = rb + 0x00010001u;
    tp.a0[jj] = rb + L - H + 0x01020102u;                    // r + rho + 257, in [3, 768]
    tp.a1[jj] = rb + H - L + 0x01020102u;                    // r - rho + 514, in [3, 768]
  }
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
// E = spread of a_0,a_2,a_4,a_6 into bytes 0,2,4,6 via one 64-bit multiply by
// 1 + 2^14 + 2^28 + 2^42; O likewise for a_1,a_3,a_5,a_7; 16-bit lanes then
// hold the pairwise sums without carries.  Verified exhaustively over all
// 2^15 windows (tests/test_swar_model.py).
template <int PARTY>
__device__ __forceinline__ void ladder_swar(uint32_t win, uint32_t& lo, uint32_t& hi) {
  constexpr uint32_t KL = 1u + (1u << 14) + (1u << 28);
  constexpr uint32_t M = 0x00FF00FFu;
  const uint32_t e = win & 0x3FFFu;
  const uint32_t o = (win >> 1) & 0x3FFFu;
  const uint32_t Elo = (e * KL) & M, Ehi = (__umulhi(e, KL) + e * 1024u) & M;
  const uint32_t Olo = (o * KL) & M, Ohi = (__umulhi(o, KL) + o * 1024u) & M;
  const uint32_t Slo = __byte_perm(Elo, Ehi, 0x5432u), Shi = Ehi >> 16;  // E >> 16: a_2,a_4,a_6,0
  uint32_t ce_lo, ce_hi, co_lo, co_hi;
  if (PARTY == 0) {  // u_i + u_{i+1} - 2 (mod 256) = v'_i - 1 for P0
    ce_lo = Elo + Olo + 0x00FE00FEu; ce_hi = Ehi + Ohi + 0x00FE00FEu;
    co_lo = Olo + Slo + 0x00FE00FEu; co_hi = Ohi + Shi + 0x00FE00FEu;
  } else {           // -(B_i + B_{i+1}) (mod 256) = v'_i - 1 for P1
    ce_lo = 0x04000400u - Elo - Olo; ce_hi = 0x04000400u - Ehi - Ohi;
    co_lo = 0x04000400u - Olo - Slo; co_hi = 0x04000400u - Ohi - Shi;
  }
  // even slots from ce (bytes 0,2), odd slots from co << 8 (bytes 1,3): c ? a : b
  lo = (ce_lo & M) | ((co_lo << 8) & ~M);
  hi = (ce_hi & M) | ((co_hi << 8) & ~M);
}

// Step 6: both Fisher-Yates phases as PRMT byte gathers.
__device__ __forceinline__ void shuffle_bytes(uint32_t& lo, uint32_t& hi, uint32_t selA, uint32_t selB) {
  const uint32_t l1 = __byte_perm(lo, hi, selA), h1 = __byte_perm(lo, hi, selA >> 16);
  lo = __byte_perm(l1, h1, selB);
  hi = __byte_perm(l1, h1, selB >> 16);
}

__device__ __forceinline__ uint32_t lane16(const uint32_t (&v)[4], int m) {
  return (m & 1) ? (v[m >> 1] >> 16) : (v[m >> 1] & 0xFFFFu);
}
__device__ __forceinline__ uint32_t mod257s(uint32_t x) {  // x < 2^18
  return x - 257u * __umulhi(x, 0xFF0100u);
}

// Steps 7-8 for one party: W_m = (c_m + 1) r_m +- rho_m (mod 257).
template <int PARTY>
__device__ __forceinline__ void mask_slots(uint32_t lo, uint32_t hi, const TapeC& tp, uint32_t (&W)[8]) {
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t c = byte_of(m < 4 ? lo : hi, m & 3);
    W[m] = mod257s(c * lane16(tp.r, m) + lane16(PARTY == 0 ? tp.a0 : tp.a1, m));
  }
}

// Steps 1-9 for both computing parties and P2 on one element; returns z.
// If W0/W1 are non-null the messages are also returned (transcript).
template <bool KEEP_W>
__device__ __forceinline__ uint32_t elem_both(uint64_t x0, uint64_t x1, const TapeC& tp, uint32_t fsh, bool fhi,
                                              uint32_t (&W0)[8], uint32_t (&W1)[8]) {
  uint32_t c_lo, c_hi, d_lo, d_hi;
  ladder_swar<0>(window_of<0>(x0, tp.t, fsh, fhi), c_lo, c_hi);
  ladder_swar<1>(window_of<1>(x1, tp.t, fsh, fhi), d_lo, d_hi);
  shuffle_bytes(c_lo, c_hi, tp.selA, tp.selB);
  shuffle_bytes(d_lo, d_hi, tp.selA, tp.selB);
  uint32_t vmin = 0xFFFFFFFFu;
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const uint32_t r = lane16(tp.r, m);
    const uint32_t w0 = mod257s(byte_of(m < 4 ? c_lo : c_hi, m & 3) * r + lane16(tp.a0, m));  // P0's message
    const uint32_t w1 = mod257s(byte_of(m < 4 ? d_lo : d_hi, m & 3) * r + lane16(tp.a1, m));  // P1's message
    if (KEEP_W) { W0[m] = w0; W1[m] = w1; }
    const uint32_t s = w0 + w1;                              // P2: w_m = W0 + W1 (mod 257)
    vmin = min(vmin, s - 257u * (s >> 8));                   // 0 iff s in {0, 257}; s <= 512
  }
  return vmin == 0u;
}

template <int PARTY>
__device__ __forceinline__ void elem_one(uint64_t x, const TapeC& tp, uint32_t fsh, bool fhi, uint32_t (&W)[8]) {
  uint32_t lo, hi;
  ladder_swar<PARTY>(window_of<PARTY>(x, tp.t, fsh, fhi), lo, hi);
  shuffle_bytes(lo, hi, tp.selA, tp.selB);
  mask_slots<PARTY>(lo, hi, tp, W);
}

}  // namespace bc
