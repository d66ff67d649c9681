// bc_fused.cu -- fused simulated three-party DReLU / ReLU (bc_drelu, bc_relu).
//
// One kernel runs P0's and P1's local phase (Alg 7 steps 1-8), P2's zero test
// and reshare (steps 9-10) and the finish (step 11, or Alg 8's Beaver
// combine) per element, with no HBM round trip for the messages: per element
// 16 B of input shares are read and 16 B of output shares written.
#include <cstdlib>

#include "bc_common.cuh"

using namespace bc;
using namespace bc::host;

namespace {

struct FusedArgs {
  const uint64_t* x0;
  const uint64_t* x1;
  uint64_t* y0;
  uint64_t* y1;
  uint64_t n, base;
  uint8_t *w0lo, *w0hi, *w1lo, *w1hi;
};

// Every stream of the fused kernels with its first-round precomputation
// (KeyPre, chacha_pre); BC_CHACHA_PRE = 0 runs the plain block function.
struct PreKeys {
  KeyPre tpa, tpb, resp, a02, b02, c02, a12, b12;
  KeyPre tri[5];  // the triple streams in the order the streamed ReLU finish consumes them: a12, a02, b02, b12, c02
};
#ifndef BC_CHACHA_PRE
#define BC_CHACHA_PRE 1
#endif
#ifndef BC_RELU_FUSED_ADDS
#define BC_RELU_FUSED_ADDS 1
#endif
#ifndef BC_RELU_PRE
#define BC_RELU_PRE 1  // the ReLU table kernel's blocks with the first-round precomputation too
#endif
#ifndef BC_RELU_STREAMED
#define BC_RELU_STREAMED 0  // 1: Alg 8's five triple blocks at ONE chacha_pre call site, each consumed before the next
#endif
// PRE: use the precomputation at this call site.  Measured (tools/variants.py):
// DReLU 0.490 -> 0.484 ms / 2^24; in round 1's SWAR ReLU kernel 0.860 -> 0.880 (the
// peeled first double round at its seven call sites cost more instruction cache than
// it saved), so k_fused_c's ReLU keeps the plain block function; the table kernels
// (k_fused_t / k_fused_tl) take it for every block (BC_RELU_PRE, ReLU 0.804 -> 0.788).
template <int R, bool PRE, bool HI0 = false>
__device__ __forceinline__ void stream_blk(const KeyPre& P, const Key& k, uint64_t label, uint64_t ctr,
                                           uint32_t (&o)[16]) {
  if (PRE && BC_CHACHA_PRE)
    chacha_pre<R, HI0>(P, ctr, o);
  else
    chacha<R>(k, ctr, label, o);
}

// ---- shared finish: Alg 7 steps 10-11, or Alg 8 (triple, e, d, Beaver combine) ----
// FULL (ell = 64): every value is already reduced mod 2^ell, the masks fold away.
// The sign (1 - 2t) is applied as a 64-bit multiply (FMA pipe) rather than as
// negate-and-select (ALU pipe, which the ChaCha rounds saturate).
template <int R, bool RELU, bool FULL, bool HI0 = false, bool STREAMED = (BC_RELU_STREAMED != 0)>
__device__ __forceinline__ void finish_group(const FusedArgs& a, const KP& kp, const Key& k02, const Key& k12,
                                             const PreKeys& pk, uint64_t i0, uint64_t j0, uint32_t cnt,
                                             uint32_t zbits, uint32_t tbits) {
  const uint64_t ym = FULL ? ~0ull : kp.ymask;
  uint64_t y0[8], y1[8];
  if (!RELU) {
    // Alg 7 step 10: P2 reshares DReLU' ([D']_0 from seed02); step 11: P0/P1 unblind.
    uint32_t Q[16];
    stream_blk<R, true, HI0>(pk.resp, k02, L_RESP, j0 >> 3, Q);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint64_t z = (zbits >> e) & 1u, t = (tbits >> e) & 1u;
      const uint64_t sgn = 1ull - 2ull * t;  // 1 - 2t (mod 2^64)
      const uint64_t q = u64_of(Q, e);       // [D']_0 (mod 2^ell)
      y0[e] = (t + sgn * q) & ym;            // t + (1-2t)[D']_0
      y1[e] = (sgn * (z - q)) & ym;          // (1-2t)[D']_1, [D']_1 = D' - [D']_0
    }
  } else if (STREAMED && BC_RELU_PRE) {
    // Alg 8 with the Beaver combine regrouped so that each triple block is consumed before the
    // next one is generated, all five at one call site (instruction cache).  With X = [x]_0 + [x]_1,
    // d = X - a, e = z - b and P = X - [a]_1 (= d + [a]_0), in Z_{2^64}:
    //   y0' = de + d[b]_0 + e[a]_0 + [c]_0   = (z - [b]_1) P - [a]_0 [b]_0 + [c]_0
    //   y1' = d[b]_1 + e[a]_1 + ab - [c]_0   = [b]_1 P + z [a]_1 + [a]_0 [b]_0 - [c]_0
    // (ring identities: the outputs are the same integers as the form below).
    uint64_t P[8], acc0[8], acc1[8];
#pragma unroll 1
    for (int s = 0; s < 5; ++s) {  // pk.tri: a12, a02, b02, b12, c02; s is uniform
      uint32_t B[16];
      chacha_pre<R, HI0>(pk.tri[s], j0 >> 3, B);
      if (s == 0) {  // [a]_1 (seed12)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const ulonglong2 v0 = load2(a.x0, i0 + 2 * h, a.n), v1 = load2(a.x1, i0 + 2 * h, a.n);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int e = 2 * h + q;
            const uint64_t a1 = u64_of(B, e);
            P[e] = ((q ? v0.y : v0.x) + (q ? v1.y : v1.x)) - a1;
            acc1[e] = a1 * (uint64_t)((zbits >> e) & 1u);  // z [a]_1
          }
        }
      } else if (s == 1) {  // [a]_0 (seed02), parked in acc0 until [b]_0 arrives
#pragma unroll
        for (int e = 0; e < 8; ++e) acc0[e] = u64_of(B, e);
      } else if (s == 2) {  // [b]_0 (seed02)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint64_t m = acc0[e] * u64_of(B, e);  // [a]_0 [b]_0
          acc0[e] = 0ull - m;
          acc1[e] += m;
        }
      } else if (s == 3) {  // [b]_1 (seed12)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint64_t b1 = u64_of(B, e);
          acc0[e] += ((uint64_t)((zbits >> e) & 1u) - b1) * P[e];
          acc1[e] += b1 * P[e];
        }
      } else {  // [c]_0 (seed02); [c]_1 = ab - [c]_0 is P2's
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint64_t c0v = u64_of(B, e);
          acc0[e] += c0v;
          acc1[e] -= c0v;
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const ulonglong2 v0 = load2(a.x0, i0 + 2 * h, a.n), v1 = load2(a.x1, i0 + 2 * h, a.n);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int e = 2 * h + q;
        const uint64_t t = (tbits >> e) & 1u;
        const uint64_t sgn = 1ull - 2ull * t;
        y0[e] = (t * (q ? v0.y : v0.x) + sgn * acc0[e]) & ym;  // t[x]_0 + (1-2t) y0'
        y1[e] = (t * (q ? v1.y : v1.x) + sgn * acc1[e]) & ym;
      }
    }
  } else {
    // Alg 8: triple from seed02 / seed12, e from P2, d opened by P0/P1, combine.
    uint64_t b0[8], b1[8], ev[8];
    {
      uint32_t Bk[16];
      stream_blk<R, BC_RELU_PRE != 0, HI0>(pk.b02, k02, L_B02, j0 >> 3, Bk);
#pragma unroll
      for (int e = 0; e < 8; ++e) b0[e] = u64_of(Bk, e);
      stream_blk<R, BC_RELU_PRE != 0, HI0>(pk.b12, k12, L_B12, j0 >> 3, Bk);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        b1[e] = u64_of(Bk, e);
#if BC_RELU_FUSED_ADDS
        b0[e] = b0[e] + b1[e];                        // b = [b]_0 + [b]_1 (P2), kept in place of [b]_0
        ev[e] = ((zbits >> e) & 1u) - b0[e];          // P2: e = DReLU' - b
#else
        ev[e] = ((zbits >> e) & 1u) - b0[e] - b1[e];  // P2: e = DReLU' - ([b]_0 + [b]_1)
#endif
      }
    }
    {
      uint32_t Ak0[16], Ak1[16];
      stream_blk<R, BC_RELU_PRE != 0, HI0>(pk.a02, k02, L_A02, j0 >> 3, Ak0);
      stream_blk<R, BC_RELU_PRE != 0, HI0>(pk.a12, k12, L_A12, j0 >> 3, Ak1);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const ulonglong2 v0 = load2(a.x0, i0 + 2 * h, a.n), v1 = load2(a.x1, i0 + 2 * h, a.n);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int e = 2 * h + s;
          const uint64_t a0 = u64_of(Ak0, e), a1 = u64_of(Ak1, e);
#if BC_RELU_FUSED_ADDS
          // the same sums with fewer separate 64-bit adds (ALU pipe, which ChaCha saturates): the
          // products' addends fold into their multiply-adds (IMAD.WIDE chains, FMA pipe).
          // b0 holds b = [b]_0 + [b]_1 (above); e + [b]_0 = DReLU' - [b]_1.
          const uint64_t av = a0 + a1;                                         // a (P2)
          const uint64_t d = ((s ? v0.y : v0.x) + (s ? v1.y : v1.x)) - av;     // opened d = x - a
          const uint64_t zb1 = ((zbits >> e) & 1u) - b1[e];                    // e + [b]_0
          y0[e] = d * zb1 + ev[e] * a0;                                        // P0: de + d[b]_0 + e[a]_0
          y1[e] = d * b1[e] + (ev[e] * a1 + av * b0[e]);                       // P1: d[b]_1 + e[a]_1 + ab
#else
          const uint64_t d = ((s ? v0.y : v0.x) - a0) + ((s ? v1.y : v1.x) - a1);  // opened d = x - a
          y0[e] = d * ev[e] + d * b0[e] + ev[e] * a0;                          // P0: de + d[b]_0 + e[a]_0
          y1[e] = d * b1[e] + ev[e] * a1 + (a0 + a1) * (b0[e] + b1[e]);        // P1: d[b]_1 + e[a]_1 + ab
#endif
        }
      }
    }
    {
      uint32_t Ck[16];
      stream_blk<R, BC_RELU_PRE != 0, HI0>(pk.c02, k02, L_C02, j0 >> 3, Ck);
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const ulonglong2 v0 = load2(a.x0, i0 + 2 * h, a.n), v1 = load2(a.x1, i0 + 2 * h, a.n);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int e = 2 * h + s;
          const uint64_t c0v = u64_of(Ck, e);
          const uint64_t t = (tbits >> e) & 1u;
          const uint64_t in0 = y0[e] + c0v;  // ... + [c]_0
          const uint64_t in1 = y1[e] - c0v;  // [c]_1 = ab - [c]_0 (P2)
          const uint64_t x0v = s ? v0.y : v0.x, x1v = s ? v1.y : v1.x;
          const uint64_t sgn = 1ull - 2ull * t;
          y0[e] = (t * x0v + sgn * in0) & ym;  // t[x] + (1-2t)(...)
          y1[e] = (t * x1v + sgn * in1) & ym;
        }
      }
    }
  }
  store8(a.y0 + i0, y0, cnt);
  store8(a.y1 + i0, y1, cnt);
}

// Compact tape (p = 257, 8 slots): per 8-element group one part-B block
// (8 B/element) and two part-A blocks (16 B/element, 4 elements each) -- 3
// ChaCha blocks per 8 elements, none shared between threads.
template <int R, bool RELU, bool TRANSCRIPT, bool FULL>
__global__ void __launch_bounds__(TPB, FUSED_MINB) k_fused_c(FusedArgs a, KP kp, Key k01, Key k02, Key k12, const __grid_constant__ PreKeys pk) {
  __shared__ uint32_t sA[2 * PERM_A], sB[2 * PERM_B];
  build_perm_tables(sA, sB);
  __syncthreads();
  const bool fhi = kp.fhi != 0;
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint32_t zbits = 0, tbits = 0;
    uint32_t Bp[16];  // part B: words 2e, 2e+1 of element e (reshare words w1, w2)
    stream_blk<R, !RELU>(pk.tpb, k01, L_TAPEB, j0 >> 3, Bp);
#pragma unroll 1
    for (int hb = 0; hb < 2; ++hb) {
      const uint64_t ib = i0 + 4 * hb;
      const ulonglong2 u0 = load2(a.x0, ib, a.n), u1 = load2(a.x1, ib, a.n);
      const ulonglong2 v0 = load2(a.x0, ib + 2, a.n), v1 = load2(a.x1, ib + 2, a.n);
      uint32_t A[16];  // part A: words 4q..4q+3 of element 4 hb + q
      stream_blk<R, !RELU>(pk.tpa, k01, L_TAPEA, (j0 >> 2) + (uint64_t)hb, A);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = 4 * hb + q;
        TapeC tp;
        decode_c<R>(A[4 * q], A[4 * q + 1], A[4 * q + 2], A[4 * q + 3], Bp[2 * q], Bp[2 * q + 1],
                    j0 + (uint64_t)e, k01, sA, sB, tp);
        const uint64_t xa = q == 0 ? u0.x : q == 1 ? u0.y : q == 2 ? v0.x : v0.y;
        const uint64_t xb = q == 0 ? u1.x : q == 1 ? u1.y : q == 2 ? v1.x : v1.y;
        uint32_t W0[8], W1[8];
        const uint32_t z = elem_both<TRANSCRIPT, !RELU>(xa, xb, tp, kp.fsh, fhi, kp.one, W0, W1);
        if (TRANSCRIPT && (uint32_t)e < cnt) {  // the P0/P1 -> P2 messages, wire format
          reinterpret_cast<uint64_t*>(a.w0lo)[i0 + e] = pack_lo(W0);
          reinterpret_cast<uint64_t*>(a.w1lo)[i0 + e] = pack_lo(W1);
          a.w0hi[i0 + e] = (uint8_t)pack_hi(W0);
          a.w1hi[i0 + e] = (uint8_t)pack_hi(W1);
        }
        zbits |= z << e;
        tbits |= tp.t << e;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) Bp[k] = Bp[k + 8];  // elements 4..7 next
    }
    finish_group<R, RELU, FULL>(a, kp, k02, k12, pk, i0, j0, cnt, zbits, tbits);
  }
}

// Compact tape, table form (bc_tables.cuh): one CTA of TPB_T threads per SM with
// the 210 KB of ladder and permutation tables in shared memory.  Same tape, same
// thread mapping and the same finish as k_fused_c.
#ifndef BC_FUSED_TABLES
#define BC_FUSED_TABLES 1  // 0: the SWAR kernel k_fused_c for the compact tape
#endif
#ifndef BC_HB_UNROLL
#define BC_HB_UNROLL 1  // the table kernel's two half-group iterations rolled (1) or unrolled (2)
#endif
constexpr int kHbUnroll = BC_HB_UNROLL;
#ifndef BC_TPB_T
#define BC_TPB_T 512  // threads of the one CTA per SM (65536 registers / TPB_T per thread)
#endif
constexpr int TPB_T = BC_TPB_T;
constexpr size_t kTabBytes = sizeof(uint32_t) * kTabWords;
__device__ constexpr CompactTables kTables{};

__device__ __forceinline__ void load_tables(uint32_t* s) {
  const uint4* g = reinterpret_cast<const uint4*>(kTables.w);
  uint4* d = reinterpret_cast<uint4*>(s);
  for (int i = threadIdx.x; i < kTabWords / 4; i += blockDim.x) d[i] = g[i];
}

template <int R, bool RELU, bool TRANSCRIPT, bool FULL, bool FHI, int MAT = BC_MATERIALIZE, bool HI0 = false>
__global__ void __launch_bounds__(TPB_T, 1) k_fused_t(FusedArgs a, KP kp, const __grid_constant__ Key k01, Key k02, Key k12, const __grid_constant__ PreKeys pk) {
  extern __shared__ uint4 smem_t[];
  uint32_t* tabs = reinterpret_cast<uint32_t*>(smem_t);
  __shared__ __align__(8) uint64_t tab_bar;
  bool tab_ready = !BC_TAB_TMA;
  if (BC_TAB_TMA) {
    if (threadIdx.x == 0) tab_bar_init(&tab_bar);
    __syncthreads();
    if (threadIdx.x == 0) tab_bulk_load(tabs, kTables.w, (uint32_t)kTabBytes, &tab_bar);
  } else {
    load_tables(tabs);
    __syncthreads();
  }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tabs);
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB_T + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB_T) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint32_t zbits = 0, tbits = 0;
    uint32_t Bp[16];  // part B: words 2e, 2e+1 of element e (reshare words w1, w2)
    stream_blk<R, !RELU || BC_RELU_PRE, HI0>(pk.tpb, k01, L_TAPEB, j0 >> 3, Bp);
#pragma unroll kHbUnroll
    for (int hb = 0; hb < 2; ++hb) {
      const uint64_t ib = i0 + 4 * hb;
      const ulonglong2 u0 = load2(a.x0, ib, a.n), u1 = load2(a.x1, ib, a.n);
      const ulonglong2 v0 = load2(a.x0, ib + 2, a.n), v1 = load2(a.x1, ib + 2, a.n);
      uint32_t A[16];  // part A: words 4q..4q+3 of element 4 hb + q
      stream_blk<R, !RELU || BC_RELU_PRE, HI0>(pk.tpa, k01, L_TAPEA, (j0 >> 2) + (uint64_t)hb, A);
      const uint32_t bit0 = 1u << (4 * hb);
      if (BC_TAB_TMA && !tab_ready) {  // the first table access of this thread: the bulk copies have landed
        tab_bar_wait(&tab_bar);
        tab_ready = true;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = 4 * hb + q;
        const uint32_t T0 = A[4 * q];
        const uint32_t t = T0 >> 31;
        const uint32_t rb[2] = {A[4 * q + 1], A[4 * q + 2]};
        const uint64_t xa = q == 0 ? u0.x : q == 1 ? u0.y : q == 2 ? v0.x : v0.y;
        const uint64_t xb = q == 0 ? u1.x : q == 1 ? u1.y : q == 2 ? v1.x : v1.y;
        uint32_t W0[8], W1[8];
#if BC_TBL_V2
        uint32_t o0[8], o1[8];
        const uint32_t ix = decode_t2<R>(T0, A[4 * q + 3], Bp[2 * q], Bp[2 * q + 1], j0 + (uint64_t)e, k01, o0, o1);
        const uint32_t z = elem_both_t2<TRANSCRIPT, FHI, MAT>(xa, xb, t, ix, rb, o0, o1, sbase, kp.fsh, kp.one, W0, W1);
#else
        uint32_t rho[8];
        const uint32_t ix = decode_t<R>(T0, A[4 * q + 3], Bp[2 * q], Bp[2 * q + 1], j0 + (uint64_t)e, k01, rho);
        const uint32_t z = elem_both_t<TRANSCRIPT, FHI>(xa, xb, t, ix, rb, rho, sbase, kp.fsh, kp.one, W0, W1);
#endif
        if (TRANSCRIPT && (uint32_t)e < cnt) {  // the P0/P1 -> P2 messages, wire format
          reinterpret_cast<uint64_t*>(a.w0lo)[i0 + e] = pack_lo(W0);
          reinterpret_cast<uint64_t*>(a.w1lo)[i0 + e] = pack_lo(W1);
          a.w0hi[i0 + e] = (uint8_t)pack_hi(W0);
          a.w1hi[i0 + e] = (uint8_t)pack_hi(W1);
        }
        const uint32_t bit = bit0 << q;
        zbits = z * bit + zbits;   // IMADs: the bit masks on the FMA pipe
        tbits = t * bit + tbits;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) Bp[k] = Bp[k + 8];  // elements 4..7 next
    }
    finish_group<R, RELU, FULL, HI0>(a, kp, k02, k12, pk, i0, j0, cnt, zbits, tbits);
  }
  if (BC_TAB_TMA && !tab_ready) tab_bar_wait(&tab_bar);  // no CTA exits with its bulk copies in flight
}

// The paper-literal domain at lx = 7 (BC_TAPE_COMPACT_LIT: w = 7, p = 131, 8 slots; pair
// tape), table form: one CTA of TPB_T threads per SM with the 186 KB of LiteralTables in
// shared memory.  Same thread mapping and finish as k_fused_w.
#ifndef BC_FUSED_LIT_TABLES
#define BC_FUSED_LIT_TABLES 1  // 0: k_fused_w<CL = true>
#endif
constexpr size_t kLitTabBytes = sizeof(uint32_t) * kLitTabWords;
__device__ constexpr LiteralTables kLitTables{};

template <int R, bool RELU, bool TRANSCRIPT, bool FULL, bool FHI, bool HI0 = false>
__global__ void __launch_bounds__(TPB_T, 1) k_fused_tl(FusedArgs a, KP kp_, const __grid_constant__ Key k01, Key k02, Key k12, const __grid_constant__ PreKeys pk) {
  const KP kp = kp_literal(kp_);
  extern __shared__ uint4 smem_t[];
  __shared__ __align__(8) uint64_t tab_bar;
  bool tab_ready = !BC_TAB_TMA;
  if (BC_TAB_TMA) {  // bulk copies (TMA) of the tables, overlapped with the first keystream blocks
    if (threadIdx.x == 0) tab_bar_init(&tab_bar);
    __syncthreads();
    if (threadIdx.x == 0) tab_bulk_load(reinterpret_cast<uint32_t*>(smem_t), kLitTables.w, (uint32_t)kLitTabBytes, &tab_bar);
  } else {
    const uint4* g = reinterpret_cast<const uint4*>(kLitTables.w);
    for (int i = threadIdx.x; i < kLitTabWords / 4; i += blockDim.x) smem_t[i] = g[i];
    __syncthreads();
  }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_t);
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB_T + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB_T) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint32_t zbits = 0, tbits = 0;
#pragma unroll 1
    for (int e2 = 0; e2 < 8; e2 += 2) {  // one seed01 block holds elements e2, e2 + 1 (j0 is a multiple of 8)
      uint32_t B[16];
      stream_blk<R, !RELU || BC_RELU_PRE, HI0>(pk.tpa, k01, L_TAPEP, (j0 + (uint64_t)e2) >> 1, B);  // bc2.tpp1
      const ulonglong2 u0 = load2(a.x0, i0 + e2, a.n), u1 = load2(a.x1, i0 + e2, a.n);
      const uint32_t bit0 = 1u << e2;
      if (BC_TAB_TMA && !tab_ready) {  // this thread's first table access
        tab_bar_wait(&tab_bar);
        tab_ready = true;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = e2 + h;
        uint32_t t, r[8], rho[8];
        const uint32_t ix = decode_pl<R>(B + 8 * h, j0 + (uint64_t)e, k01, kp, t, r, rho);
        uint32_t W0[8], W1[8];
        const uint32_t z = elem_both_tl<TRANSCRIPT, FHI>(h ? u0.y : u0.x, h ? u1.y : u1.x, t, ix, r, rho, sbase,
                                                         kp.fsh, W0, W1);
        if (TRANSCRIPT && (uint32_t)e < cnt) {  // the P0/P1 -> P2 messages, wire format
          reinterpret_cast<uint64_t*>(a.w0lo)[i0 + e] = pack_lo(W0);
          reinterpret_cast<uint64_t*>(a.w1lo)[i0 + e] = pack_lo(W1);
          a.w0hi[i0 + e] = (uint8_t)pack_hi(W0);
          a.w1hi[i0 + e] = (uint8_t)pack_hi(W1);
        }
        const uint32_t bit = bit0 << h;
        zbits = z * bit + zbits;
        tbits = t * bit + tbits;
      }
    }
    finish_group<R, RELU, FULL, HI0>(a, kp, k02, k12, pk, i0, j0, cnt, zbits, tbits);
  }
  if (BC_TAB_TMA && !tab_ready) tab_bar_wait(&tab_bar);  // no CTA exits with its bulk copies in flight
}

// Pair tape (every lx <= 7 domain but the compact one: p <= 131, 3..8 slots): one
// seed01 block per two elements (bc2.tpp1, 32 B each).
template <int R, bool RELU, bool CL>
__global__ void __launch_bounds__(TPB, 2) k_fused_w(FusedArgs a, KP kp_, Key k01, Key k02, Key k12, const __grid_constant__ PreKeys pk) {
  const KP kp = CL ? kp_literal(kp_) : kp_;
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint32_t zbits = 0, tbits = 0;
#pragma unroll 1
    for (int e2 = 0; e2 < 8; e2 += 2) {  // one seed01 block holds elements e2, e2 + 1 (j0 is a multiple of 8)
      uint32_t B[16];
      stream_blk<R, !RELU>(pk.tpa, k01, L_TAPEP, (j0 + (uint64_t)e2) >> 1, B);  // pk.tpa: bc2.tpp1
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // static offsets into B keep it in registers
      const int e = e2 + h;
      const uint64_t xa = (uint32_t)e < cnt ? __ldg(a.x0 + i0 + e) : 0ull;
      const uint64_t xb = (uint32_t)e < cnt ? __ldg(a.x1 + i0 + e) : 0ull;
      Tape tp;
      decode_pair<R>(B + 8 * h, j0 + e, k01, kp, tp);
      uint32_t W0[8], W1[8];
      party_W_rt<0>(xa, kp, tp, W0);
      party_W_rt<1>(xb, kp, tp, W1);
      zbits |= zero_test(W0, W1, kp.p, kp.S) << e;
      tbits |= tp.t << e;
      if (a.w0lo != nullptr && (uint32_t)e < cnt) {
        reinterpret_cast<uint64_t*>(a.w0lo)[i0 + e] = pack_lo(W0);
        reinterpret_cast<uint64_t*>(a.w1lo)[i0 + e] = pack_lo(W1);
        a.w0hi[i0 + e] = (uint8_t)pack_hi(W0);
        a.w1hi[i0 + e] = (uint8_t)pack_hi(W1);
      }
    }
    }
    finish_group<R, RELU, false>(a, kp, k02, k12, pk, i0, j0, cnt, zbits, tbits);
  }
}

// Large tape (lx >= 8, up to 32 slots, p < 2^33): 7 seed01 blocks per element (bc2.tpL2),
// the 8 elements of a group in sequence, then the shared finish.
constexpr int TPB_L = TPB_LARGE;
#ifndef BC_LARGE_PRE
#define BC_LARGE_PRE 1  // the large tape's 7 blocks through chacha_pre (pk.tpa = (seed01, bc2.tpL2))
#endif
#ifndef BC_LARGE_RELU_MINB
#define BC_LARGE_RELU_MINB 5  // resident CTAs the large-tape ReLU kernel is compiled for (register cap 102; measured 7.91 -> 7.70 ms, 4 CTAs: 8.00)
#endif
#ifndef BC_LARGE_RELU_STREAMED
#define BC_LARGE_RELU_STREAMED 0  // 1: the large-tape ReLU kernel's finish with the streamed Beaver blocks (137 registers, was 124)
#endif
#ifndef BC_LARGE_MINB
#define BC_LARGE_MINB 1  // resident CTAs per SM the large-tape kernel is compiled for (register cap)
#endif

template <int R, bool RELU, bool TRANSCRIPT, bool HI0 = false, bool W32 = false, bool L31 = false>
__global__ void __launch_bounds__(TPB_L, RELU ? BC_LARGE_RELU_MINB : BC_LARGE_MINB) k_fused_l(FusedArgs a, KP kp, KPL kl, Key k01, Key k02, Key k12,
                                                                  const __grid_constant__ PreKeys pk) {
  __shared__ uint32_t sidx[kIdxWords * TPB_L];
  __shared__ uint32_t sstg[LARGE_STG_ROWS * TPB_L];
  __shared__ uint32_t magic[33], hlim[33];
  large_tables(magic, hlim);
  __syncthreads();
  LargeIdx* idx = reinterpret_cast<LargeIdx*>(sidx + threadIdx.x);
  uint32_t* stg = sstg + threadIdx.x;
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB_L + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB_L) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint32_t zbits = 0, tbits = 0;
#pragma unroll 1
    for (uint32_t e = 0; e < cnt; ++e) {
      const uint64_t i = i0 + e;
      uint64_t* w0 = TRANSCRIPT ? reinterpret_cast<uint64_t*>(a.w0lo) + i * kl.S : nullptr;
      uint64_t* w1 = TRANSCRIPT ? reinterpret_cast<uint64_t*>(a.w1lo) + i * kl.S : nullptr;
      const uint32_t r =
          elem_large<R, TRANSCRIPT, TPB_L, BC_LARGE_PRE != 0, HI0, W32, RELU, L31>(__ldg(a.x0 + i), __ldg(a.x1 + i), j0 + e, k01, kl, idx,
                                                                    stg, magic, hlim, w0, w1, &pk.tpa);
      zbits |= (r & 1u) << e;
      tbits |= (r >> 1) << e;
    }
    finish_group<R, RELU, false, HI0, BC_LARGE_RELU_STREAMED != 0>(a, kp, k02, k12, pk, i0, j0, cnt, zbits, tbits);
  }
}

// ---- Bicoptor-1 as Bicoptor 2.0 describes it (NEXT #4; readings C32-C34) ----------
// SecureML truncation (u_i in Z_{2^ell}), recursive sums, no modulo switch, odd
// 64-bit masks and 64-bit reshares: 3 seed01 blocks per element (bc1.tape).
constexpr uint64_t L_TAPE1 = lbl("bc1.tape");
constexpr uint64_t L_FB1 = lbl("bc1.fbk1");

template <int R>
__device__ __noinline__ uint32_t fallback_b1(uint64_t j, Key key, uint32_t lim) {
  uint32_t B[16];
  for (uint32_t k = 0;; ++k) {
    if ((k & 15u) == 0) chacha<R>(key, j * 256 + (k >> 4), L_FB1, B);
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if ((uint32_t)i == (k & 15u)) w = B[i];
    const uint32_t v = w & 0x7FFFFFFFu;
    if (v < lim) return v;
  }
}

template <int R, bool TRANSCRIPT>
__global__ void __launch_bounds__(TPB_L) k_fused_b1(FusedArgs a, KP kp, Key k01, Key k02, Key k12, const __grid_constant__ PreKeys pk) {
  __shared__ uint64_t sv[2 * 8 * TPB_L];  // [party][slot][thread]
  const uint32_t tid = threadIdx.x, S = kp.S;
  const uint64_t ym = kp.ymask;
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB_L + tid; g < ngroups; g += (uint64_t)gridDim.x * TPB_L) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint32_t zbits = 0, tbits = 0;
#pragma unroll 1
    for (uint32_t e = 0; e < cnt; ++e) {
      const uint64_t j = j0 + e, i = i0 + e;
      uint64_t r[8], rho[8];
      uint32_t t, idx;
      {
        uint32_t B[16];
        chacha<R>(k01, 3 * j, L_TAPE1, B);             // words 0..15: t|idx, r_0..r_6
        t = B[0] >> 31;
        idx = B[0] & 0x7FFFFFFFu;
#pragma unroll
        for (int m = 0; m < 7; ++m) r[m] = (uint64_t)B[2 + 2 * m] | ((uint64_t)B[3 + 2 * m] << 32);
        chacha<R>(k01, 3 * j + 1, L_TAPE1, B);         // words 16..31: r_7, rho_0..rho_6
        r[7] = (uint64_t)B[0] | ((uint64_t)B[1] << 32);
#pragma unroll
        for (int m = 0; m < 7; ++m) rho[m] = (uint64_t)B[2 + 2 * m] | ((uint64_t)B[3 + 2 * m] << 32);
        chacha<R>(k01, 3 * j + 2, L_TAPE1, B);         // words 32, 33: rho_7
        rho[7] = (uint64_t)B[0] | ((uint64_t)B[1] << 32);
      }
      if (idx >= kp.perm_lim) idx = fallback_b1<R>(j, k01, kp.perm_lim);
      // step 6: Fisher-Yates nibble selector (same digits as the pair tape)
      uint32_t sel = 0x76543210u;
      for (uint32_t m = S - 1; m >= 1; --m) {
        const uint32_t k = idx % (m + 1);
        idx /= (m + 1);
        const uint32_t aa = (sel >> (4 * m)) & 15u, bb = (sel >> (4 * k)) & 15u, d = aa ^ bb;
        sel ^= (d << (4 * m)) ^ (d << (4 * k));
      }
      // steps 1-4: blind, Alg 1 truncations u_i = trc(s, f+i) in Z_{2^ell}, recursive sums
      const uint64_t x0v = __ldg(a.x0 + i), x1v = __ldg(a.x1 + i);
      const uint64_t s0 = (t ? 0ull - x0v : x0v) & ym;
      const uint64_t n1 = (t ? x1v : 0ull - x1v) & ym;  // -s1 mod 2^ell
      uint64_t acc0 = 0, acc1 = 0;
#pragma unroll
      for (int q = 7; q >= 0; --q) {
        if ((uint32_t)q < S) {
          acc0 += s0 >> (kp.f + q);                    // P0: cut(s0, f+q)
          acc1 -= n1 >> (kp.f + q);                    // P1: -cut(-s1, f+q)
          sv[(0 * 8 + q) * TPB_L + tid] = acc0 - 1ull; // v_q, P0 carries the -1
          sv[(1 * 8 + q) * TPB_L + tid] = acc1;
        }
      }
      // steps 6-9: shuffle, mask (odd r), reshare, P2's zero test, all mod 2^ell
      uint32_t z = 0;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        if ((uint32_t)m < S) {
          const uint32_t src = (sel >> (4 * m)) & 15u;
          const uint64_t rm = r[m] | 1ull;
          const uint64_t W0 = (sv[src * TPB_L + tid] * rm + rho[m]) & ym;
          const uint64_t W1 = (sv[(8 + src) * TPB_L + tid] * rm - rho[m]) & ym;
          if (TRANSCRIPT) {
            reinterpret_cast<uint64_t*>(a.w0lo)[i * S + m] = W0;
            reinterpret_cast<uint64_t*>(a.w1lo)[i * S + m] = W1;
          }
          z |= ((W0 + W1) & ym) == 0 ? 1u : 0u;
        }
      }
      zbits |= z << e;
      tbits |= t << e;
    }
    finish_group<R, false, false>(a, kp, k02, k12, pk, i0, j0, cnt, zbits, tbits);
  }
}

// BICOPTOR_MATERIALIZE=2 in the environment (a measurement knob, read per call; bench.py's
// "materialize2" leg): the compact table kernel at ell = 64 reduces BOTH computing parties'
// messages to their wire values W in [0, 257) and P2 adds wire values, as the transcript
// path and the party kernels do, instead of testing P0's W0 + P1's
// congruent x1.  Same results; this times the difference.
bool wire_values_mode() {
  const char* e = std::getenv("BICOPTOR_MATERIALIZE");
  return e && e[0] == '2';
}

template <bool RELU>
int fused(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n, uint64_t base,
          const bc_params* prm, const bc_seeds* seeds, const bc_transcript* tr, void* stream) {
  const int rc = check_params(prm);
  if (rc) return rc;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if (!x0 || !x1 || !y0 || !y1 || !seeds) return BC_EINVAL;
  if (!aligned16(x0) || !aligned16(x1) || !aligned16(y0) || !aligned16(y1) || (base & 7)) return BC_EALIGN;
  if (!index_range_ok(base, n)) return BC_ERANGE;  // global indices j < BC_MAX_INDEX
  const size_t nb = n * 8;
  if (overlap(y0, nb, y1, nb) || overlap(y0, nb, x0, nb) || overlap(y0, nb, x1, nb) || overlap(y1, nb, x0, nb) ||
      overlap(y1, nb, x1, nb))
    return BC_EALIAS;
  FusedArgs a{x0, x1, y0, y1, (uint64_t)n, base, nullptr, nullptr, nullptr, nullptr};
  const bool large = prm->tape == BC_TAPE_LARGE;
  if (tr && large) {  // W planes as uint64_t[n][slots]
    if (!tr->w0_lo || !tr->w1_lo || tr->w0_hi || tr->w1_hi) return BC_EINVAL;
    if (!aligned8(tr->w0_lo) || !aligned8(tr->w1_lo)) return BC_EALIGN;
    const size_t wb = n * prm->slots * 8;
    if (overlap(tr->w0_lo, wb, tr->w1_lo, wb) || overlap(tr->w0_lo, wb, x0, nb) || overlap(tr->w0_lo, wb, x1, nb) ||
        overlap(tr->w1_lo, wb, x0, nb) || overlap(tr->w1_lo, wb, x1, nb) || overlap(tr->w0_lo, wb, y0, nb) ||
        overlap(tr->w0_lo, wb, y1, nb) || overlap(tr->w1_lo, wb, y0, nb) || overlap(tr->w1_lo, wb, y1, nb))
      return BC_EALIAS;
    a.w0lo = tr->w0_lo;
    a.w1lo = tr->w1_lo;
  } else if (tr) {  // the transcript is all-or-nothing
    if (!tr->w0_lo || !tr->w0_hi || !tr->w1_lo || !tr->w1_hi) return BC_EINVAL;
    if (!aligned8(tr->w0_lo) || !aligned8(tr->w1_lo)) return BC_EALIGN;
    a.w0lo = tr->w0_lo;
    a.w0hi = tr->w0_hi;
    a.w1lo = tr->w1_lo;
    a.w1hi = tr->w1_hi;
  }
  const KP kp = make_kp(prm);
  const Key k01 = make_key(seeds->s01), k02 = make_key(seeds->s02), k12 = make_key(seeds->s12);
  const uint64_t tape_a = prm->tape == BC_TAPE_COMPACT ? L_TAPEA : prm->tape == BC_TAPE_LARGE ? L_TAPEL : L_TAPEP;
  const PreKeys pk{make_keypre(seeds->s01, tape_a), make_keypre(seeds->s01, L_TAPEB),
                   make_keypre(seeds->s02, L_RESP),  make_keypre(seeds->s02, L_A02),
                   make_keypre(seeds->s02, L_B02),   make_keypre(seeds->s02, L_C02),
                   make_keypre(seeds->s12, L_A12),   make_keypre(seeds->s12, L_B12),
                   {make_keypre(seeds->s12, L_A12), make_keypre(seeds->s02, L_A02), make_keypre(seeds->s02, L_B02),
                    make_keypre(seeds->s12, L_B12), make_keypre(seeds->s02, L_C02)}};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t ngroups = (n + 7) / 8;
  return dispatch_rounds(prm->rounds, [&](auto Rc) {
    constexpr int R = decltype(Rc)::value;
    if (large) {
      const KPL kl = make_kpl(prm);
      auto fn = tr ? k_fused_l<R, RELU, true> : k_fused_l<R, RELU, false>;
      if (!tr) {
        const bool hi0 = base + n <= (1ull << 32) / 7;  // every tape counter 7j + b below 2^32
        if (kl.w == 32)  // p = 2^32 + 15: the pseudo-Mersenne slot arithmetic
          fn = hi0 ? k_fused_l<R, RELU, false, true, true> : k_fused_l<R, RELU, false, false, true>;
        else if (kl.w == 31 && kl.S == 32 && kl.p == P31)  // the paper-literal full precision, p = 2^31 + 11
          fn = hi0 ? k_fused_l<R, RELU, false, true, false, true> : k_fused_l<R, RELU, false, false, false, true>;
        else if (hi0)
          fn = k_fused_l<R, RELU, false, true>;
      }
      fn<<<grid_for((const void*)fn, ngroups, TPB_L), TPB_L, 0, st>>>(a, kp, kl, k01, k02, k12, pk);
    } else if (prm->tape == BC_TAPE_COMPACT && BC_FUSED_TABLES) {
      const bool fhi = kp.fhi != 0;
      auto fn = tr ? (fhi ? k_fused_t<R, RELU, true, false, true> : k_fused_t<R, RELU, true, false, false>)
                   : prm->ell == 64 ? (fhi ? k_fused_t<R, RELU, false, true, true> : k_fused_t<R, RELU, false, true, false>)
                                    : (fhi ? k_fused_t<R, RELU, false, false, true> : k_fused_t<R, RELU, false, false, false>);
      if (!tr && prm->ell == 64 && !fhi) {
        // every keystream counter below 2^32 (part A: j/4, part B and the response: j/8): the
        // first round's column 1 is precomputed on the host as well (chacha_pre<R, true>)
        const bool hi0 = base + n <= (1ull << 34);
        if (wire_values_mode())  // measurement knob: both wire values reduced
          fn = hi0 ? k_fused_t<R, RELU, false, true, false, 2, true> : k_fused_t<R, RELU, false, true, false, 2>;
        else if (hi0)
          fn = k_fused_t<R, RELU, false, true, false, BC_MATERIALIZE, true>;
      }
      const int rc = allow_smem((const void*)fn, kTabBytes);
      if (rc) return rc;
      fn<<<grid_for((const void*)fn, ngroups, TPB_T, kTabBytes), TPB_T, kTabBytes, st>>>(a, kp, k01, k02, k12, pk);
    } else if (prm->tape == BC_TAPE_COMPACT) {
      auto fn = tr ? k_fused_c<R, RELU, true, false>
                   : (prm->ell == 64 ? k_fused_c<R, RELU, false, true> : k_fused_c<R, RELU, false, false>);
      fn<<<grid_for((const void*)fn, ngroups), TPB, 0, st>>>(a, kp, k01, k02, k12, pk);
    } else if (prm->tape == BC_TAPE_COMPACT_LIT && BC_FUSED_LIT_TABLES) {
      const bool fhi = kp.fhi != 0;
      auto fn = tr ? (fhi ? k_fused_tl<R, RELU, true, false, true> : k_fused_tl<R, RELU, true, false, false>)
                   : prm->ell == 64 ? (fhi ? k_fused_tl<R, RELU, false, true, true> : k_fused_tl<R, RELU, false, true, false>)
                                    : (fhi ? k_fused_tl<R, RELU, false, false, true> : k_fused_tl<R, RELU, false, false, false>);
      if (!tr && prm->ell == 64 && !fhi && base + n <= (1ull << 33))  // pair-tape counters j/2 below 2^32
        fn = k_fused_tl<R, RELU, false, true, false, true>;
      const int rc = allow_smem((const void*)fn, kLitTabBytes);
      if (rc) return rc;
      fn<<<grid_for((const void*)fn, ngroups, TPB_T, kLitTabBytes), TPB_T, kLitTabBytes, st>>>(a, kp, k01, k02, k12, pk);
    } else {
      auto fn = prm->tape == BC_TAPE_COMPACT_LIT ? k_fused_w<R, RELU, true> : k_fused_w<R, RELU, false>;
      fn<<<grid_for((const void*)fn, ngroups), TPB, 0, st>>>(a, kp, k01, k02, k12, pk);
    }
    return check_launch();
  });
}

int drelu_b1(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n, uint64_t base,
             const bc_params* prm, const bc_seeds* seeds, const bc_transcript* tr, void* stream) {
  const int rc = check_params(prm);
  if (rc) return rc;
  if (prm->slots > 8) return BC_EINVAL;
  if (n == 0) return BC_OK;
  if (!x0 || !x1 || !y0 || !y1 || !seeds) return BC_EINVAL;
  if (!aligned16(x0) || !aligned16(x1) || !aligned16(y0) || !aligned16(y1) || (base & 7)) return BC_EALIGN;
  if (!index_range_ok(base, n)) return BC_ERANGE;  // global indices j < BC_MAX_INDEX
  const size_t nb = n * 8;
  if (overlap(y0, nb, y1, nb) || overlap(y0, nb, x0, nb) || overlap(y0, nb, x1, nb) || overlap(y1, nb, x0, nb) ||
      overlap(y1, nb, x1, nb))
    return BC_EALIAS;
  FusedArgs a{x0, x1, y0, y1, (uint64_t)n, base, nullptr, nullptr, nullptr, nullptr};
  if (tr) {  // W planes as uint64_t[n][slots]
    if (!tr->w0_lo || !tr->w1_lo || tr->w0_hi || tr->w1_hi) return BC_EINVAL;
    if (!aligned8(tr->w0_lo) || !aligned8(tr->w1_lo)) return BC_EALIGN;
    const size_t wb = n * prm->slots * 8;
    if (overlap(tr->w0_lo, wb, tr->w1_lo, wb) || overlap(tr->w0_lo, wb, x0, nb) || overlap(tr->w0_lo, wb, x1, nb) ||
        overlap(tr->w1_lo, wb, x0, nb) || overlap(tr->w1_lo, wb, x1, nb) || overlap(tr->w0_lo, wb, y0, nb) ||
        overlap(tr->w0_lo, wb, y1, nb) || overlap(tr->w1_lo, wb, y0, nb) || overlap(tr->w1_lo, wb, y1, nb))
      return BC_EALIAS;
    a.w0lo = tr->w0_lo;
    a.w1lo = tr->w1_lo;
  }
  KP kp = make_kp(prm);
  const uint32_t fact = [&] { uint32_t f = 1; for (uint32_t i = 2; i <= prm->slots; ++i) f *= i; return f; }();
  kp.perm_lim = (uint32_t)((0x80000000ull / fact) * fact);
  const Key k01 = make_key(seeds->s01), k02 = make_key(seeds->s02), k12 = make_key(seeds->s12);
  const PreKeys pk{make_keypre(seeds->s01, L_TAPEA), make_keypre(seeds->s01, L_TAPEB),
                   make_keypre(seeds->s02, L_RESP),  make_keypre(seeds->s02, L_A02),
                   make_keypre(seeds->s02, L_B02),   make_keypre(seeds->s02, L_C02),
                   make_keypre(seeds->s12, L_A12),   make_keypre(seeds->s12, L_B12),
                   {make_keypre(seeds->s12, L_A12), make_keypre(seeds->s02, L_A02), make_keypre(seeds->s02, L_B02),
                    make_keypre(seeds->s12, L_B12), make_keypre(seeds->s02, L_C02)}};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return dispatch_rounds(prm->rounds, [&](auto Rc) {
    constexpr int R = decltype(Rc)::value;
    auto fn = tr ? k_fused_b1<R, true> : k_fused_b1<R, false>;
    fn<<<grid_for((const void*)fn, (n + 7) / 8, TPB_L), TPB_L, 0, st>>>(a, kp, k01, k02, k12, pk);
    return check_launch();
  });
}

}  // namespace

extern "C" {

int bc_drelu_b1(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n, uint64_t elem_base,
                const bc_params* prm, const bc_seeds* seeds, const bc_transcript* tr, void* stream) {
  return drelu_b1(x0, x1, y0, y1, n, elem_base, prm, seeds, tr, stream);
}

int bc_drelu(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n, uint64_t elem_base,
             const bc_params* prm, const bc_seeds* seeds, const bc_transcript* tr, void* stream) {
  return fused<false>(x0, x1, y0, y1, n, elem_base, prm, seeds, tr, stream);
}

int bc_relu(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n, uint64_t elem_base,
            const bc_params* prm, const bc_seeds* seeds, const bc_transcript* tr, void* stream) {
  return fused<true>(x0, x1, y0, y1, n, elem_base, prm, seeds, tr, stream);
}

}  // extern "C"
