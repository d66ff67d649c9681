// bc_rss.cu -- RSS variant (Alg 9; RSS ReLU by secret
// multiplication): bc_drelu_rss, bc_relu_rss, all three parties
// simulated on one GPU in one fused kernel.
//
// Replicated shares: x = x_0 + x_1 + x_2 mod 2^ell, party P_i holds (x_i, x_{i+1}).
// Per 8-element group a thread
//   1. expands the group's preprocessing streams (reading C25) --
//      seed012: alpha_0..2, [s]_1; seed12: [s]_2; seed2: the bit s; the
//      multiplication zero-sharing F02, F01, F12 (and a second one for ReLU) --
//      one ChaCha block per stream, staged in shared memory (transposed, one
//      column per thread: conflict-free);
//   2. runs Alg 7 steps 1-9 on the bridged 2-of-2 sharing (P0: x_0 + x_1,
//      P1: x_2; online step 1) with the compact-tape path of the UBL kernel;
//   3. P2: DReLU'' = s xor DReLU'; all parties: [DReLU] = DReLU'' + [u] -
//      2 DReLU''[u] with [u] = [s] + [t] - 2[s][t] (preprocessing step 3);
//   4. ReLU: the secret multiplication [x][DReLU] (reading C26).
#include "bc_common.cuh"

using namespace bc;
using namespace bc::host;

namespace {

#ifndef BC_TPB_RSS
#define BC_TPB_RSS 128
#endif
// threads per CTA: the staged preprocessing keystream is 576 B per thread (DReLU),
// so the CTA size sets how many CTAs fit in shared memory
constexpr int TPB_RSS = BC_TPB_RSS;

constexpr uint64_t L_RA0 = lbl("bc2.ra00"), L_RA1 = lbl("bc2.ra01"), L_RA2 = lbl("bc2.ra02");  // seed012: alpha_k
constexpr uint64_t L_RS01 = lbl("bc2.rs01");   // seed012: [s]_1
constexpr uint64_t L_RS12 = lbl("bc2.rs12");   // seed12:  [s]_2
constexpr uint64_t L_RS2B = lbl("bc2.rs2b");   // seed2:   s (bit 0)
constexpr uint64_t L_RM02 = lbl("bc2.rm02"), L_RM01 = lbl("bc2.rm01"), L_RM12 = lbl("bc2.rm12");  // [s][t]
constexpr uint64_t L_RN02 = lbl("bc2.rn02"), L_RN01 = lbl("bc2.rn01"), L_RN12 = lbl("bc2.rn12");  // [x][DReLU]

// stream index -> (key, label); streams 9..11 only for ReLU
enum { S_A0, S_A1, S_A2, S_S1, S_S2, S_SB, S_M02, S_M01, S_M12, S_N02, S_N01, S_N12, NS_MAX };

struct RssArgs {
  const uint64_t *x0, *x1, *x2;
  uint64_t *y0, *y1, *y2;
  uint64_t n, base;
};

struct RssKeys {
  Key k01, k02, k12, k012, k2;
  KeyPre pre[NS_MAX];    // every preprocessing stream's (key, label) with chacha_pre's first-round columns
  KeyPre tpa, tpb;       // the compact tape's two seed01 streams
};

#ifndef BC_RSS_PRE
#define BC_RSS_PRE 1  // every block through chacha_pre at one call site (stream s selects K.pre[s])
#endif
template <int R>
__device__ __forceinline__ void stream_block(const RssKeys& K, int s, uint64_t blk, uint32_t (&B)[16]) {
  switch (s) {
    case S_A0: chacha<R>(K.k012, blk, L_RA0, B); break;
    case S_A1: chacha<R>(K.k012, blk, L_RA1, B); break;
    case S_A2: chacha<R>(K.k012, blk, L_RA2, B); break;
    case S_S1: chacha<R>(K.k012, blk, L_RS01, B); break;
    case S_S2: chacha<R>(K.k12, blk, L_RS12, B); break;
    case S_SB: chacha<R>(K.k2, blk, L_RS2B, B); break;
    case S_M02: chacha<R>(K.k02, blk, L_RM02, B); break;
    case S_M01: chacha<R>(K.k01, blk, L_RM01, B); break;
    case S_M12: chacha<R>(K.k12, blk, L_RM12, B); break;
    case S_N02: chacha<R>(K.k02, blk, L_RN02, B); break;
    case S_N01: chacha<R>(K.k01, blk, L_RN01, B); break;
    default: chacha<R>(K.k12, blk, L_RN12, B); break;
  }
}

// RSS product component i (reading C26): a_i b_i + a_i b_{i+1} + a_{i+1} b_i + g_i
__device__ __forceinline__ void rss_mul(const uint64_t (&a)[3], const uint64_t (&b)[3], const uint64_t (&g)[3],
                                        uint64_t (&z)[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int k = (i + 1) % 3;
    z[i] = a[i] * b[i] + a[i] * b[k] + a[k] * b[i] + g[i];
  }
}

template <int R, bool RELU, bool HI0 = false>
__global__ void __launch_bounds__(TPB_RSS) k_fused_rss(RssArgs a, KP kp, const __grid_constant__ RssKeys K) {
  constexpr int NS = RELU ? 12 : 9;
  __shared__ uint32_t sA[2 * PERM_A], sB[2 * PERM_B];
  extern __shared__ uint32_t ks[];  // [NS][16][TPB_RSS]
  build_perm_tables(sA, sB);
  __syncthreads();
  const bool fhi = kp.fhi != 0;
  const uint32_t tid = threadIdx.x;
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB_RSS + tid; g < ngroups; g += (uint64_t)gridDim.x * TPB_RSS) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    // ---- 1. preprocessing streams of the group -> shared memory ---------------
#pragma unroll 1
    for (int s = 0; s < NS; ++s) {
      uint32_t B[16];
      if (BC_RSS_PRE)
        chacha_pre<R, HI0>(K.pre[s], j0 >> 3, B);  // s is warp-uniform: K.pre[s] is a uniform constant-bank read
      else
        stream_block<R>(K, s, j0 >> 3, B);
#pragma unroll
      for (int w = 0; w < 16; ++w) ks[(s * 16 + w) * TPB_RSS + tid] = B[w];
    }
    // ---- 2. Alg 7 steps 1-9 on the bridged sharing (P0: x_0 + x_1, P1: x_2) ---
    uint32_t zbits = 0, tbits = 0;
    uint32_t Bp[16];
    if (BC_RSS_PRE)
      chacha_pre<R, HI0>(K.tpb, j0 >> 3, Bp);
    else
      chacha<R>(K.k01, j0 >> 3, L_TAPEB, Bp);
#pragma unroll 1
    for (int hb = 0; hb < 2; ++hb) {
      const uint64_t ib = i0 + 4 * hb;
      const ulonglong2 p0 = load2(a.x0, ib, a.n), p1 = load2(a.x1, ib, a.n), p2 = load2(a.x2, ib, a.n);
      const ulonglong2 q0 = load2(a.x0, ib + 2, a.n), q1 = load2(a.x1, ib + 2, a.n), q2 = load2(a.x2, ib + 2, a.n);
      uint32_t A[16];
      if (BC_RSS_PRE)
        chacha_pre<R, HI0>(K.tpa, (j0 >> 2) + (uint64_t)hb, A);
      else
        chacha<R>(K.k01, (j0 >> 2) + (uint64_t)hb, L_TAPEA, A);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = 4 * hb + q;
        TapeC tp;
        decode_c<R>(A[4 * q], A[4 * q + 1], A[4 * q + 2], A[4 * q + 3], Bp[2 * q], Bp[2 * q + 1],
                    j0 + (uint64_t)e, K.k01, sA, sB, tp);
        const uint64_t xa = q == 0 ? p0.x + p1.x : q == 1 ? p0.y + p1.y : q == 2 ? q0.x + q1.x : q0.y + q1.y;
        const uint64_t xb = q == 0 ? p2.x : q == 1 ? p2.y : q == 2 ? q2.x : q2.y;
        uint32_t W0[8], W1[8];
        zbits |= elem_both<false>(xa, xb, tp, kp.fsh, fhi, kp.one, W0, W1) << e;
        tbits |= tp.t << e;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) Bp[k] = Bp[k + 8];
    }
    // ---- 3. preprocessing algebra, P2's DReLU'', the output components -------
#pragma unroll 1
    for (int e = 0; e < 8; ++e) {
      auto rd = [&](int s) {
        return (uint64_t)ks[(s * 16 + 2 * e) * TPB_RSS + tid] | ((uint64_t)ks[(s * 16 + 2 * e + 1) * TPB_RSS + tid] << 32);
      };
      const uint64_t t = (tbits >> e) & 1u;
      const uint64_t al0 = rd(S_A0), al1 = rd(S_A1), al2 = rd(S_A2);
      const uint64_t tsh[3] = {al0 - al2, al1 - al0 + t, al2 - al1};          // [t]_1 = [beta]_1 + t
      const uint64_t s1 = rd(S_S1), s2 = rd(S_S2), sb = rd(S_SB) & 1u;
      const uint64_t ssh[3] = {sb - s1 - s2, s1, s2};                          // [s]_0 = s - [s]_1 - [s]_2
      const uint64_t f02 = rd(S_M02), f01 = rd(S_M01), f12 = rd(S_M12);
      const uint64_t gz[3] = {f02 - f01, f01 - f12, f12 - f02};                // zero sharing
      uint64_t st[3];
      rss_mul(ssh, tsh, gz, st);                                               // [s][t]
      const uint64_t d2 = ((zbits >> e) & 1u) ^ sb;                            // P2: DReLU'' = s xor DReLU'
      uint64_t y[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint64_t u = ssh[k] + tsh[k] - 2u * st[k];                       // [s xor t]
        y[k] = u - 2u * d2 * u + (k == 0 ? d2 : 0ull);                         // D'' + [u] - 2 D''[u]
      }
      if (RELU) {                                                              // [x][DReLU(x)]
        const uint64_t i = i0 + e;
        const uint64_t xv[3] = {(uint32_t)e < cnt ? a.x0[i] : 0ull, (uint32_t)e < cnt ? a.x1[i] : 0ull,
                                (uint32_t)e < cnt ? a.x2[i] : 0ull};
        const uint64_t n02 = rd(S_N02), n01 = rd(S_N01), n12 = rd(S_N12);
        const uint64_t g2[3] = {n02 - n01, n01 - n12, n12 - n02};
        uint64_t r[3];
        rss_mul(xv, y, g2, r);
        y[0] = r[0]; y[1] = r[1]; y[2] = r[2];
      }
      if ((uint32_t)e < cnt) {
        a.y0[i0 + e] = y[0] & kp.ymask;
        a.y1[i0 + e] = y[1] & kp.ymask;
        a.y2[i0 + e] = y[2] & kp.ymask;
      }
    }
  }
}

// ---- table form with the preprocessing streamed (BC_RSS_TABLES) ---------------------------
// Step 2 as the UBL table kernel k_fused_t (one CTA of 512 threads per SM, the 210 KB of
// ladder and 8! selector tables in shared memory), then the preprocessing blocks one at a
// time at ONE chacha_pre call site, each consumed before the next is generated -- nothing is
// staged, so the 576 B/thread of k_fused_rss's keystream staging (12% warps active) is gone.
// The algebra of step 3 is regrouped so that a block's values enter linear accumulators
// (ring identities in Z_{2^64}; same outputs).  With sigma = s, k1 = 2[s]_1, k2 = 2([s]_2 - s):
//   u_0 = (s - [s]_1 - [s]_2) + t (k1 + k2) + a_0 (1 - k1) + a_1 (k1 + k2) - a_2 (1 + k2) - 2 (F02 - F01)
//   u_1 = [s]_1 + t (1 - 2[s]_2 - k1) + a_0 (k1 + 2[s]_2 - 1) + a_1 (1 - 2[s]_2) - a_2 k1 - 2 (F01 - F12)
//   u_2 = u - u_0 - u_1,  u = s + t - 2 s t   (the components of [s xor t], reading C26's product)
// (a_k = alpha_k; from tsh = (a0 - a2, a1 - a0 + t, a2 - a1), ssh = (s - [s]_1 - [s]_2, [s]_1, [s]_2)
// and u_k = ssh_k + tsh_k - 2 st_k).  Streams in the order SB, S1, S2, A0, A1, A2, M02, M01, M12
// (ReLU: then N02, N01, N12 into the product components r_0, r_1; r_2 = X Y - r_0 - r_1).
// Measured (2^24, ms, tools/variants.py): DReLU R20 1.2306 (k_fused_rss) vs 1.2331 (this kernel),
// ReLU 1.566 vs 1.624, R8 0.674 vs 0.741: twice the resident warps (25% instead of 12%) buy
// nothing -- the ALU pipe, not latency, bounds both -- and the ReLU accumulators spill.  Off.
#ifndef BC_RSS_TABLES
#define BC_RSS_TABLES 0  // 1: this kernel; 0: k_fused_rss above
#endif
constexpr int TPB_RT = 512;
constexpr size_t kTabBytesR = sizeof(uint32_t) * kTabWords;
__device__ constexpr CompactTables kTablesR{};

template <int R, bool RELU, bool FHI, bool HI0>
__global__ void __launch_bounds__(TPB_RT, 1) k_fused_rss_t(RssArgs a, KP kp, const __grid_constant__ RssKeys K) {
  constexpr int NS = RELU ? 12 : 9;
  extern __shared__ uint4 smem_r[];
  uint32_t* tabs = reinterpret_cast<uint32_t*>(smem_r);
  __shared__ __align__(8) uint64_t tab_bar;
  bool tab_ready = !BC_TAB_TMA;
  if (BC_TAB_TMA) {
    if (threadIdx.x == 0) tab_bar_init(&tab_bar);
    __syncthreads();
    if (threadIdx.x == 0) tab_bulk_load(tabs, kTablesR.w, (uint32_t)kTabBytesR, &tab_bar);
  } else {
    const uint4* g = reinterpret_cast<const uint4*>(kTablesR.w);
    for (int i = threadIdx.x; i < kTabWords / 4; i += blockDim.x) smem_r[i] = g[i];
    __syncthreads();
  }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tabs);
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB_RT + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB_RT) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    // ---- 2. Alg 7 steps 1-9 on the bridged sharing (P0: x_0 + x_1, P1: x_2) ---
    uint32_t zbits = 0, tbits = 0;
    {
      uint32_t Bp[16];
      chacha_pre<R, HI0>(K.tpb, j0 >> 3, Bp);
#pragma unroll 1
      for (int hb = 0; hb < 2; ++hb) {
        const uint64_t ib = i0 + 4 * hb;
        const ulonglong2 p0 = load2(a.x0, ib, a.n), p1 = load2(a.x1, ib, a.n), p2 = load2(a.x2, ib, a.n);
        const ulonglong2 q0 = load2(a.x0, ib + 2, a.n), q1 = load2(a.x1, ib + 2, a.n), q2 = load2(a.x2, ib + 2, a.n);
        uint32_t A[16];
        chacha_pre<R, HI0>(K.tpa, (j0 >> 2) + (uint64_t)hb, A);
        if (BC_TAB_TMA && !tab_ready) {
          tab_bar_wait(&tab_bar);
          tab_ready = true;
        }
        const uint32_t bit0 = 1u << (4 * hb);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int e = 4 * hb + q;
          const uint32_t T0 = A[4 * q];
          const uint32_t t = T0 >> 31;
          const uint32_t rb[2] = {A[4 * q + 1], A[4 * q + 2]};
          const uint64_t xa = q == 0 ? p0.x + p1.x : q == 1 ? p0.y + p1.y : q == 2 ? q0.x + q1.x : q0.y + q1.y;
          const uint64_t xb = q == 0 ? p2.x : q == 1 ? p2.y : q == 2 ? q2.x : q2.y;
          uint32_t o0[8], o1[8], W0[8], W1[8];
          const uint32_t ix = decode_t2<R>(T0, A[4 * q + 3], Bp[2 * q], Bp[2 * q + 1], j0 + (uint64_t)e, K.k01, o0, o1);
          const uint32_t z = elem_both_t2<false, FHI>(xa, xb, t, ix, rb, o0, o1, sbase, kp.fsh, kp.one, W0, W1);
          const uint32_t bit = bit0 << q;
          zbits = z * bit + zbits;
          tbits = t * bit + tbits;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) Bp[k] = Bp[k + 8];
      }
    }
    // ---- 3. the preprocessing streamed into the accumulators (see above) --------
    uint32_t sbits = 0;
    uint64_t s1v[8], s2v[8], U0[8], U1[8];
#pragma unroll 1
    for (int s = 0; s < NS; ++s) {
      const int st = s == 0 ? S_SB : s <= 2 ? S_S1 + (s - 1) : s <= 5 ? S_A0 + (s - 3) : s;  // uniform
      uint32_t B[16];
      chacha_pre<R, HI0>(K.pre[st], j0 >> 3, B);
      if (s == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) sbits |= (B[2 * e] & 1u) << e;                   // s (seed2)
      } else if (s == 1) {
#pragma unroll
        for (int e = 0; e < 8; ++e) s1v[e] = u64_of(B, e);                          // [s]_1
      } else if (s == 2) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          s2v[e] = u64_of(B, e);                                                     // [s]_2
          const uint64_t sg = (sbits >> e) & 1u, t = (tbits >> e) & 1u;
          const uint64_t k1 = 2u * s1v[e], k2 = 2u * (s2v[e] - sg);
          U0[e] = (sg - s1v[e] - s2v[e]) + t * (k1 + k2);
          U1[e] = s1v[e] + t * (1u - 2u * s2v[e] - k1);
        }
      } else if (s <= 5) {  // alpha_0, alpha_1, alpha_2
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint64_t al = u64_of(B, e), sg = (sbits >> e) & 1u;
          const uint64_t k1 = 2u * s1v[e], k2 = 2u * (s2v[e] - sg), s2x2 = 2u * s2v[e];
          if (s == 3) {
            U0[e] += al * (1u - k1);
            U1[e] += al * (k1 + s2x2 - 1u);
          } else if (s == 4) {
            U0[e] += al * (k1 + k2);
            U1[e] += al * (1u - s2x2);
          } else {
            U0[e] -= al * (1u + k2);
            U1[e] -= al * k1;
          }
        }
      } else if (s <= 8) {  // the zero sharing of [s][t]: F02, F01, F12
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint64_t f2 = 2u * u64_of(B, e);
          if (s == 6) U0[e] -= f2;
          if (s == 7) { U0[e] += f2; U1[e] -= f2; }
          if (s == 8) U1[e] += f2;
        }
        if (RELU && s == 8) {  // y = [DReLU] components, then the product components r_0, r_1
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const ulonglong2 v0 = load2(a.x0, i0 + 2 * h, a.n), v1 = load2(a.x1, i0 + 2 * h, a.n),
                             v2 = load2(a.x2, i0 + 2 * h, a.n);
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
              const int e = 2 * h + qq;
              const uint64_t sg = (sbits >> e) & 1u, t = (tbits >> e) & 1u;
              const uint64_t d2 = ((zbits >> e) & 1u) ^ sg, mm = 1u - 2u * d2;
              const uint64_t u = sg + t - 2u * sg * t;
              const uint64_t y0 = U0[e] * mm + d2, y1 = U1[e] * mm, y2 = (u - U0[e] - U1[e]) * mm;
              const uint64_t x0 = qq ? v0.y : v0.x, x1 = qq ? v1.y : v1.x, x2 = qq ? v2.y : v2.x;
              U0[e] = x0 * (y0 + y1) + x1 * y0;                                         // r_0 without g
              U1[e] = x1 * (y1 + y2) + x2 * y1;                                         // r_1 without g
            }
          }
        }
      } else {  // ReLU: the zero sharing of [x][DReLU]: N02, N01, N12
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint64_t nv = u64_of(B, e);
          if (s == 9) U0[e] += nv;
          if (s == 10) { U0[e] -= nv; U1[e] += nv; }
          if (s == 11) U1[e] -= nv;
        }
      }
    }
    uint64_t y0[8], y1[8], y2[8];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      ulonglong2 v0{}, v1{}, v2{};
      if (RELU) {
        v0 = load2(a.x0, i0 + 2 * h, a.n);
        v1 = load2(a.x1, i0 + 2 * h, a.n);
        v2 = load2(a.x2, i0 + 2 * h, a.n);
      }
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const int e = 2 * h + qq;
        const uint64_t sg = (sbits >> e) & 1u, t = (tbits >> e) & 1u;
        const uint64_t d2 = ((zbits >> e) & 1u) ^ sg, mm = 1u - 2u * d2;
        const uint64_t u = sg + t - 2u * sg * t;
        if (RELU) {
          const uint64_t X = (qq ? v0.y : v0.x) + (qq ? v1.y : v1.x) + (qq ? v2.y : v2.x);
          const uint64_t Y = u * mm + d2;                                                // DReLU(x)
          y0[e] = U0[e] & kp.ymask;
          y1[e] = U1[e] & kp.ymask;
          y2[e] = (X * Y - U0[e] - U1[e]) & kp.ymask;                                    // sum = X Y
        } else {
          y0[e] = (U0[e] * mm + d2) & kp.ymask;                                          // D'' + [u] - 2 D''[u]
          y1[e] = (U1[e] * mm) & kp.ymask;
          y2[e] = ((u - U0[e] - U1[e]) * mm) & kp.ymask;
        }
      }
    }
    store8(a.y0 + i0, y0, cnt);
    store8(a.y1 + i0, y1, cnt);
    store8(a.y2 + i0, y2, cnt);
  }
  if (BC_TAB_TMA && !tab_ready) tab_bar_wait(&tab_bar);
}

template <bool RELU>
int fused_rss(const uint64_t* x0, const uint64_t* x1, const uint64_t* x2, uint64_t* y0, uint64_t* y1, uint64_t* y2,
              size_t n, uint64_t base, const bc_params* prm, const bc_seeds* seeds, const uint8_t* s012,
              const uint8_t* s2, void* stream) {
  const int rc = check_params(prm);
  if (rc) return rc;
  if (prm->tape != BC_TAPE_COMPACT) return BC_EINVAL;  // RSS path: compact tape (p = 257, 8 slots) only
  if (n == 0) return BC_OK;
  if (!x0 || !x1 || !x2 || !y0 || !y1 || !y2 || !seeds || !s012 || !s2) return BC_EINVAL;
  if (!aligned16(x0) || !aligned16(x1) || !aligned16(x2) || !aligned16(y0) || !aligned16(y1) || !aligned16(y2) ||
      (base & 7))
    return BC_EALIGN;
  if (!index_range_ok(base, n)) return BC_ERANGE;  // global indices j < BC_MAX_INDEX
  const size_t nb = n * 8;
  const void* ins[3] = {x0, x1, x2};
  const void* outs[3] = {y0, y1, y2};
  for (int i = 0; i < 3; ++i) {
    for (int k = 0; k < 3; ++k)
      if (overlap(outs[i], nb, ins[k], nb)) return BC_EALIAS;
    for (int k = i + 1; k < 3; ++k)
      if (overlap(outs[i], nb, outs[k], nb)) return BC_EALIAS;
  }
  RssArgs a{x0, x1, x2, y0, y1, y2, (uint64_t)n, base};
  const KP kp = make_kp(prm);
  RssKeys K{make_key(seeds->s01), make_key(seeds->s02), make_key(seeds->s12), make_key(s012), make_key(s2), {}, {}, {}};
  {
    const uint8_t* ks[NS_MAX] = {s012, s012, s012, s012, seeds->s12, s2, seeds->s02, seeds->s01, seeds->s12,
                                 seeds->s02, seeds->s01, seeds->s12};
    const uint64_t ls[NS_MAX] = {L_RA0, L_RA1, L_RA2, L_RS01, L_RS12, L_RS2B, L_RM02, L_RM01, L_RM12,
                                 L_RN02, L_RN01, L_RN12};
    for (int s = 0; s < NS_MAX; ++s) K.pre[s] = make_keypre(ks[s], ls[s]);
    K.tpa = make_keypre(seeds->s01, L_TAPEA);
    K.tpb = make_keypre(seeds->s01, L_TAPEB);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t ngroups = (n + 7) / 8;
  const size_t smem = (size_t)(RELU ? 12 : 9) * 16 * TPB_RSS * sizeof(uint32_t);
  return dispatch_rounds(prm->rounds, [&](auto Rc) {
    constexpr int R = decltype(Rc)::value;
    if constexpr (BC_RSS_TABLES != 0) {
      const bool fhi = kp.fhi != 0, hi0 = base + n <= (1ull << 34);
      auto fn = fhi ? (hi0 ? k_fused_rss_t<R, RELU, true, true> : k_fused_rss_t<R, RELU, true, false>)
                    : (hi0 ? k_fused_rss_t<R, RELU, false, true> : k_fused_rss_t<R, RELU, false, false>);
      const int rc = allow_smem((const void*)fn, kTabBytesR);
      if (rc) return rc;
      fn<<<grid_for((const void*)fn, ngroups, TPB_RT, kTabBytesR), TPB_RT, kTabBytesR, st>>>(a, kp, K);
      return check_launch();
    }
    // every counter (j/8, j/4 + 1) below 2^32: the first round's column 1 is precomputed too
    auto fn = base + n <= (1ull << 34) ? k_fused_rss<R, RELU, true> : k_fused_rss<R, RELU, false>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, TPB_RSS, smem);
    const uint64_t want = (ngroups + TPB_RSS - 1) / TPB_RSS;
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)std::max(1, sms * occ)));
    fn<<<grid, TPB_RSS, smem, st>>>(a, kp, K);
    return check_launch();
  });
}

}  // namespace

extern "C" {

int bc_drelu_rss(const uint64_t* x0, const uint64_t* x1, const uint64_t* x2, uint64_t* y0, uint64_t* y1, uint64_t* y2,
                 size_t n, uint64_t elem_base, const bc_params* prm, const bc_seeds* seeds, const uint8_t seed012[32],
                 const uint8_t seed2[32], void* stream) {
  return fused_rss<false>(x0, x1, x2, y0, y1, y2, n, elem_base, prm, seeds, seed012, seed2, stream);
}

int bc_relu_rss(const uint64_t* x0, const uint64_t* x1, const uint64_t* x2, uint64_t* y0, uint64_t* y1, uint64_t* y2,
                size_t n, uint64_t elem_base, const bc_params* prm, const bc_seeds* seeds, const uint8_t seed012[32],
                const uint8_t seed2[32], void* stream) {
  return fused_rss<true>(x0, x1, x2, y0, y1, y2, n, elem_base, prm, seeds, seed012, seed2, stream);
}

}  // extern "C"
