// bc_party.cu -- party-separated phases of Alg 7 / Alg 8: send (P0, P1),
// helper (P2), finish (P0, P1).  Each party runs its phase on its own device.
// The message buffers are whatever the caller passes: staging buffers it then
// moves (NCCL send/recv, party.py) or the receiving party's inbox mapped into
// this process (peer.py), in which case the kernel's stores are the transfer.
#include "bc_common.cuh"

using namespace bc;
using namespace bc::host;

namespace {

struct SendArgs {
  const uint64_t* x;
  uint8_t* lo;
  uint8_t* hi;
  uint8_t* tbits;
  uint64_t* dshare;
  uint64_t* dpeer;  // nullable: second destination of [d]_b (the other computing party's inbox)
  uint64_t* y0;     // nullable (DReLU, P0): P0's output share, computed in the same kernel
  uint64_t n, base;
};

// Alg 7 steps 10-11 for P0 inside its send kernel (the transport in which P0
// derives [D']_0 from seed02 itself, reading C12): y0 = t + (1-2t) q.
template <int R>
__device__ __forceinline__ void send_finish_p0(const SendArgs& a, const KP& kp, const Key& k02, uint64_t i0,
                                               uint64_t j0, uint32_t cnt, uint32_t tb) {
  uint32_t Q[16];
  chacha<R>(k02, j0 >> 3, L_RESP, Q);
  uint64_t y[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint64_t t = (tb >> e) & 1u;
    y[e] = (t + (1ull - 2ull * t) * u64_of(Q, e)) & kp.ymask;
  }
  store8(a.y0 + i0, y, cnt);
}

__device__ __forceinline__ void store_msg(const SendArgs& a, const KP& kp, const Key& ktr, uint64_t g, uint64_t i0,
                                          uint64_t j0, uint32_t cnt, const uint64_t (&lo)[8], uint64_t hi,
                                          uint32_t tb, int party, bool relu);

// Alg 8 step 4 (first half): [d]_b = [x]_b - [a]_b for the group's 8
// elements, stored locally and (peer transport) into the other party's inbox.
template <int R, int PARTY>
__device__ __forceinline__ void send_dshare(const SendArgs& a, const KP& kp, const Key& ktr, uint64_t i0, uint64_t j0,
                                            uint32_t cnt) {
  uint32_t Ak[16];
  chacha<R>(ktr, j0 >> 3, PARTY == 0 ? L_A02 : L_A12, Ak);
  uint64_t x[8], d[8];
  load8(a.x + i0, x, cnt);
#pragma unroll
  for (int e = 0; e < 8; ++e) d[e] = (x[e] - u64_of(Ak, e)) & kp.ymask;
  store8(a.dshare + i0, d, cnt);
  if (a.dpeer) store8(a.dpeer + i0, d, cnt);  // the opening of d, stored straight into the peer
}

// Alg 7 steps 1-8 (and Alg 8's [d]_b) for one computing party, compact tape.
template <int R, int PARTY, bool RELU>
__global__ void __launch_bounds__(TPB, 2) k_send_c(SendArgs a, KP kp, Key k01, Key ktr) {
  __shared__ uint32_t sA[2 * PERM_A], sB[2 * PERM_B];
  build_perm_tables(sA, sB);
  __syncthreads();
  const bool fhi = kp.fhi != 0;
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint64_t lo[8];
    uint32_t tb = 0;
    uint64_t hi = 0;
    uint32_t Bp[16];
    chacha<R>(k01, j0 >> 3, L_TAPEB, Bp);
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const ulonglong2 u = load2(a.x, i0 + 4 * hb, a.n), v = load2(a.x, i0 + 4 * hb + 2, a.n);
      uint32_t A[16];
      chacha<R>(k01, (j0 >> 2) + (uint64_t)hb, L_TAPEA, A);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = 4 * hb + q;
        TapeC tp;
        decode_c<R>(A[4 * q], A[4 * q + 1], A[4 * q + 2], A[4 * q + 3], Bp[8 * hb + 2 * q], Bp[8 * hb + 2 * q + 1],
                    j0 + (uint64_t)e, k01, sA, sB, tp);
        uint32_t W[8];
        elem_one<PARTY, BC_ADD_FMA_SEND != 0>(q == 0 ? u.x : q == 1 ? u.y : q == 2 ? v.x : v.y, tp, kp.fsh, fhi, W, kp.one);
        lo[e] = pack_lo(W);
        hi |= (uint64_t)pack_hi(W) << (8 * e);
        tb |= tp.t << e;
      }
    }
    store_msg(a, kp, ktr, g, i0, j0, cnt, lo, hi, tb, PARTY, false);
    if (RELU) send_dshare<R, PARTY>(a, kp, ktr, i0, j0, cnt);
    if (!RELU && PARTY == 0 && a.y0) send_finish_p0<R>(a, kp, ktr, i0, j0, cnt, tb);
  }
}

// Compact tape, table form (as the fused k_fused_t): one CTA of TPB_ST threads per SM with the
// 210 KB of ladder and 8! selector tables in shared memory, the V2 slot arithmetic, and every
// keystream block through chacha_pre (HI0: every counter of the launch below 2^32).
#ifndef BC_SEND_TABLES
#define BC_SEND_TABLES 1  // 0: the SWAR kernel k_send_c
#endif
constexpr int TPB_ST = 512;
constexpr size_t kSendTabBytes = sizeof(uint32_t) * kTabWords;
__device__ constexpr CompactTables kSendTables{};

struct SendPre {
  KeyPre tpa, tpb;  // seed01: compact tape parts A and B
  KeyPre tra;       // ReLU: the party's [a]_b stream (seed02 bc2.ta02 for P0, seed12 bc2.ta12 for P1)
  KeyPre resp;      // DReLU, P0 with y0: seed02 bc2.resp
};

template <int R, int PARTY, bool RELU, bool FHI, bool HI0>
__global__ void __launch_bounds__(TPB_ST, 1) k_send_t(SendArgs a, KP kp, const __grid_constant__ Key k01, Key ktr,
                                                       const __grid_constant__ SendPre sp) {
  extern __shared__ uint4 smem_st[];
  __shared__ __align__(8) uint64_t tab_bar;
  bool tab_ready = !BC_TAB_TMA;
  if (BC_TAB_TMA) {  // bulk copies (TMA) of the tables, overlapped with the first keystream blocks
    if (threadIdx.x == 0) tab_bar_init(&tab_bar);
    __syncthreads();
    if (threadIdx.x == 0) tab_bulk_load(reinterpret_cast<uint32_t*>(smem_st), kSendTables.w, (uint32_t)kSendTabBytes, &tab_bar);
  } else {
    const uint4* g = reinterpret_cast<const uint4*>(kSendTables.w);
    for (int i = threadIdx.x; i < kTabWords / 4; i += blockDim.x) smem_st[i] = g[i];
    __syncthreads();
  }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem_st);
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB_ST + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB_ST) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint32_t tb = 0;
    uint64_t hi = 0;
    uint32_t Bp[16];
    chacha_pre<R, HI0>(sp.tpb, j0 >> 3, Bp);
#pragma unroll 1
    for (int hb = 0; hb < 2; ++hb) {
      const ulonglong2 u = load2(a.x, i0 + 4 * hb, a.n), v = load2(a.x, i0 + 4 * hb + 2, a.n);
      uint32_t A[16];
      chacha_pre<R, HI0>(sp.tpa, (j0 >> 2) + (uint64_t)hb, A);
      uint64_t lo[4];  // the half group's low-byte planes, stored at the end of the iteration
      if (BC_TAB_TMA && !tab_ready) {  // this thread's first table access
        tab_bar_wait(&tab_bar);
        tab_ready = true;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = 4 * hb + q;
        const uint32_t t = A[4 * q] >> 31;
        const uint32_t rb[2] = {A[4 * q + 1], A[4 * q + 2]};
        uint32_t o0[8], o1[8], W[8];
        const uint32_t ix = decode_t2<R>(A[4 * q], A[4 * q + 3], Bp[2 * q], Bp[2 * q + 1], j0 + (uint64_t)e, k01, o0, o1);
        elem_one_t2<PARTY, FHI>(q == 0 ? u.x : q == 1 ? u.y : q == 2 ? v.x : v.y, t, ix, rb, PARTY == 0 ? o0 : o1,
                                sbase, kp.fsh, W);
        lo[q] = pack_lo(W);
        hi |= (uint64_t)pack_hi(W) << (8 * e);
        tb |= t << e;
      }
      uint64_t* lop = reinterpret_cast<uint64_t*>(a.lo) + i0 + 4 * hb;
      const uint32_t c4 = cnt > 4u * hb ? min(4u, cnt - 4u * hb) : 0u;
      if (c4 == 4) {
        reinterpret_cast<ulonglong2*>(lop)[0] = make_ulonglong2(lo[0], lo[1]);
        reinterpret_cast<ulonglong2*>(lop)[1] = make_ulonglong2(lo[2], lo[3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if ((uint32_t)q < c4) lop[q] = lo[q];
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) Bp[k] = Bp[k + 8];  // elements 4..7 next
    }
    if (a.hi) {  // the high-bit plane (bit 8 of each W_m) and the blinding bits, as store_msg
      if (cnt == 8) *reinterpret_cast<uint64_t*>(a.hi + i0) = hi;
      else
        for (uint32_t e = 0; e < cnt; ++e) a.hi[i0 + e] = (uint8_t)(hi >> (8 * e));
    }
    if (a.tbits) a.tbits[g] = (uint8_t)(tb & ((1u << cnt) - 1u));
    if (RELU) {  // Alg 8 step 4: [d]_b = [x]_b - [a]_b (as send_dshare, block through chacha_pre)
      uint32_t Ak[16];
      chacha_pre<R, HI0>(sp.tra, j0 >> 3, Ak);
      uint64_t x[8], d[8];
      load8(a.x + i0, x, cnt);
#pragma unroll
      for (int e = 0; e < 8; ++e) d[e] = (x[e] - u64_of(Ak, e)) & kp.ymask;
      store8(a.dshare + i0, d, cnt);
      if (a.dpeer) store8(a.dpeer + i0, d, cnt);
    }
    if (!RELU && PARTY == 0 && a.y0) {  // Alg 7 steps 10-11 for P0 (as send_finish_p0)
      uint32_t Q[16];
      chacha_pre<R, HI0>(sp.resp, j0 >> 3, Q);
      uint64_t y[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint64_t t = (tb >> e) & 1u;
        y[e] = (t + (1ull - 2ull * t) * u64_of(Q, e)) & kp.ymask;
      }
      store8(a.y0 + i0, y, cnt);
    }
  }
  if (BC_TAB_TMA && !tab_ready) tab_bar_wait(&tab_bar);  // no CTA exits with its bulk copies in flight
}

// Pair tape (one seed01 block per two elements).
template <int R, int PARTY, bool RELU, bool CL>
__global__ void __launch_bounds__(TPB, 2) k_send_w(SendArgs a, KP kp_, Key k01, Key ktr) {
  const KP kp = CL ? kp_literal(kp_) : kp_;
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint64_t lo[8];
    uint32_t tb = 0;
    uint64_t hi = 0;
#pragma unroll 1
    for (int e2 = 0; e2 < 8; e2 += 2) {  // one seed01 block holds elements e2, e2 + 1 (j0 is a multiple of 8)
      uint32_t B[16];
      chacha<R>(k01, (j0 + (uint64_t)e2) >> 1, L_TAPEP, B);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // static offsets into B keep it in registers
      const int e = e2 + h;
      const uint64_t xv = (uint32_t)e < cnt ? __ldg(a.x + i0 + e) : 0ull;
      Tape tp;
      decode_pair<R>(B + 8 * h, j0 + e, k01, kp, tp);
      uint32_t W[8];
      party_W_rt<PARTY>(xv, kp, tp, W);
      const uint64_t l = pack_lo(W);
      const uint64_t hbyte = pack_hi(W);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k == e) lo[k] = l;
      hi |= hbyte << (8 * e);
      tb |= tp.t << e;
    }
    }
    store_msg(a, kp, ktr, g, i0, j0, cnt, lo, hi, tb, PARTY, false);
    if (RELU) send_dshare<R, PARTY>(a, kp, ktr, i0, j0, cnt);
    if (!RELU && PARTY == 0 && a.y0) send_finish_p0<R>(a, kp, ktr, i0, j0, cnt, tb);
  }
}

// Large tape (lx >= 8: up to 32 slots, p < 2^33).  Wire format, slot-major:
// lo = uint32_t[S][n] (word m of element i at lo[m n + i]: the low 32 bits of
// W_m), hi = uint32_t[n] (bit m = bit 32 of W_m; NULL when p < 2^32): 33 S
// bits per element, 132 B at lx = 31 guard.  A warp owns 256 consecutive
// elements: first lane l computes elements base + 32 e + l (e = 0..7), so the
// stores of slot m are 128 coalesced bytes (over NVLink in the peer
// transport) and the blinding bits come out of one ballot per 32 elements;
// then (ReLU) lane l computes [d]_b for its group of 8 (send_dshare).
template <int R, int PARTY, bool RELU, bool W32 = false, bool HI0 = false, bool L31 = false>
__global__ void __launch_bounds__(TPB_LARGE) k_send_l(SendArgs a, KP kp, KPL kl, Key k01, Key ktr,
                                                      const __grid_constant__ KeyPre tpl) {
  __shared__ uint32_t sidx[kIdxWords * TPB_LARGE];
  __shared__ uint32_t sstg[LARGE_STG_ROWS * TPB_LARGE];
  __shared__ uint32_t magic[33], hlim[33];
  large_tables(magic, hlim);
  __syncthreads();
  LargeIdx* idx = reinterpret_cast<LargeIdx*>(sidx + threadIdx.x);
  uint32_t* stg = sstg + threadIdx.x;
  uint32_t* lo = reinterpret_cast<uint32_t*>(a.lo);
  uint32_t* hi = reinterpret_cast<uint32_t*>(a.hi);
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t ngroups = (a.n + 7) >> 3, nbytes = ngroups;
  const uint64_t warps = (uint64_t)gridDim.x * (TPB_LARGE / 32);
  for (uint64_t wb = ((uint64_t)blockIdx.x * (TPB_LARGE / 32) + threadIdx.x / 32) * 256; wb < a.n;
       wb += warps * 256) {
    uint32_t tgroup = 0;
#pragma unroll 1
    for (uint32_t e = 0; e < 8; ++e) {
      const uint64_t i = wb + 32 * e + lane;
      uint32_t tb = 0;
      if (i < a.n) {
        const uint64_t r = elem_large_party<R, PARTY, TPB_LARGE, W32, true, HI0, L31>(__ldg(a.x + i), a.base + i, k01, kl, idx, stg,
                                                                 magic, hlim, lo + i, a.n, &tpl);
        if (hi) hi[i] = (uint32_t)r;
        tb = (uint32_t)(r >> 32);
      }
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, tb != 0u);  // t of elements wb + 32 e + 0..31
      const uint64_t byte = (wb + 32 * e) / 8 + lane;
      if (lane < 4 && byte < nbytes && a.tbits) a.tbits[byte] = (uint8_t)(bal >> (8 * lane));
      if ((lane >> 2) == e) tgroup = (bal >> (8 * (lane & 3u))) & 0xFFu;  // t bits of lane's group
    }
    if (!RELU && PARTY == 0 && a.y0) {
      const uint64_t g = wb / 8 + lane;
      if (g < ngroups) {
        const uint64_t i0 = g << 3;
        send_finish_p0<R>(a, kp, ktr, i0, a.base + i0, (uint32_t)min((uint64_t)8, a.n - i0), tgroup);
      }
    }
    if (RELU) {
      const uint64_t g = wb / 8 + lane;
      if (g < ngroups) {
        const uint64_t i0 = g << 3;
        send_dshare<R, PARTY>(a, kp, ktr, i0, a.base + i0, (uint32_t)min((uint64_t)8, a.n - i0));
      }
    }
  }
}

__device__ __forceinline__ void store_msg(const SendArgs& a, const KP& kp, const Key& ktr, uint64_t g, uint64_t i0,
                                          uint64_t j0, uint32_t cnt, const uint64_t (&lo)[8], uint64_t hi,
                                          uint32_t tb, int party, bool relu) {
  store8(reinterpret_cast<uint64_t*>(a.lo) + i0, lo, cnt);
  if (a.hi) {
    if (cnt == 8) *reinterpret_cast<uint64_t*>(a.hi + i0) = hi;
    else
      for (uint32_t e = 0; e < cnt; ++e) a.hi[i0 + e] = (uint8_t)(hi >> (8 * e));
  }
  if (a.tbits) a.tbits[g] = (uint8_t)(tb & ((1u << cnt) - 1u));
}

struct HelperArgs {
  const uint8_t *lo0, *hi0, *lo1, *hi1;
  uint64_t* out0;   // DReLU: resp0 (nullable)   ReLU: e
  uint64_t* out0b;  // nullable: second destination of out0 (ReLU: e to P1 as well as P0)
  uint64_t* out1;   // DReLU: resp1              ReLU: c1 (nullable)
  uint64_t n, base;
};

// The seed02 / seed12 streams of the helper and finish phases with chacha_pre's first-round
// precomputation (host: make_keypre; only the streams of the seeds the caller passed are set).
struct StreamPre {
  KeyPre resp, b02, b12, a02, a12, c02;
};

// P2's response for a group with zero-test bits zbits: Alg 7 step 10 ([D']_0
// from seed02, [D']_1 = DReLU' - [D']_0), or Alg 8 steps 2-3 (e = DReLU' - b and
// [c]_1 = ab - [c]_0 from the triple seeds).
template <int R, bool RELU, bool HI0>
__device__ __forceinline__ void helper_respond(const HelperArgs& a, const KP& kp, const StreamPre& sp,
                                               uint64_t i0, uint64_t j0, uint32_t cnt, uint32_t zbits) {
  uint64_t o0[8], o1[8];
  if (!RELU) {
    uint32_t Q[16];
    chacha_pre<R, HI0>(sp.resp, j0 >> 3, Q);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint64_t q = u64_of(Q, e) & kp.ymask;
      o0[e] = q;
      o1[e] = (((zbits >> e) & 1u) - q) & kp.ymask;
    }
  } else {
    uint32_t Bk0[16], Bk1[16];
    chacha_pre<R, HI0>(sp.b02, j0 >> 3, Bk0);
    chacha_pre<R, HI0>(sp.b12, j0 >> 3, Bk1);
    uint64_t bsum[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      bsum[e] = u64_of(Bk0, e) + u64_of(Bk1, e);
      o0[e] = (((zbits >> e) & 1u) - bsum[e]) & kp.ymask;  // e = DReLU' - b
    }
    if (a.out1) {  // [c]_1 = ([a]_0 + [a]_1)([b]_0 + [b]_1) - [c]_0
      uint32_t Ak0[16], Ak1[16];
      chacha_pre<R, HI0>(sp.a02, j0 >> 3, Ak0);
      chacha_pre<R, HI0>(sp.a12, j0 >> 3, Ak1);
#pragma unroll
      for (int e = 0; e < 8; ++e) o1[e] = (u64_of(Ak0, e) + u64_of(Ak1, e)) * bsum[e];
      uint32_t Ck[16];
      chacha_pre<R, HI0>(sp.c02, j0 >> 3, Ck);
#pragma unroll
      for (int e = 0; e < 8; ++e) o1[e] = (o1[e] - u64_of(Ck, e)) & kp.ymask;
    }
  }
  if (a.out0) store8(a.out0 + i0, o0, cnt);
  if (a.out0b) store8(a.out0b + i0, o0, cnt);
  if (a.out1) store8(a.out1 + i0, o1, cnt);
}

// P2: Alg 7 steps 9-10, or Alg 8 steps 2-3 with the triple's [c]_1.
template <int R, bool RELU, bool HI0 = false>
__global__ void __launch_bounds__(TPB, 2) k_helper(HelperArgs a, KP kp, const __grid_constant__ StreamPre sp) {
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint64_t l0[8], l1[8];
    load8(reinterpret_cast<const uint64_t*>(a.lo0) + i0, l0, cnt);
    load8(reinterpret_cast<const uint64_t*>(a.lo1) + i0, l1, cnt);
    const uint64_t h0 = load_hi8(a.hi0, i0, cnt), h1 = load_hi8(a.hi1, i0, cnt);
    uint32_t zbits = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {  // step 9: reconstruct w_m, look for a zero
      uint32_t W0[8], W1[8];
      unpack_W(l0[e], (uint32_t)(h0 >> (8 * e)) & 0xFFu, W0);
      unpack_W(l1[e], (uint32_t)(h1 >> (8 * e)) & 0xFFu, W1);
      zbits |= zero_test(W0, W1, kp.p, kp.S) << e;
    }
    helper_respond<R, RELU, HI0>(a, kp, sp, i0, j0, cnt, zbits);
  }
}

// P2 on the large-tape wire format (slot-major, see k_send_l).  A warp owns
// 256 consecutive elements: lane l tests elements base + 32 e + l, reading
// slot m of both messages as 128 coalesced bytes per warp, 8 slots' loads in
// flight at a time; a ballot per 32 elements hands each lane the DReLU' byte
// of its own group of 8, for which it then answers (helper_respond).
#ifndef BC_HELPER_L_MINB
#define BC_HELPER_L_MINB 2
#endif
template <int R, bool RELU, bool HI0 = false>
__global__ void __launch_bounds__(TPB, BC_HELPER_L_MINB) k_helper_l(HelperArgs a, KP kp, KPL kl,
                                                                    const __grid_constant__ StreamPre sp) {
  const uint32_t* lo0 = reinterpret_cast<const uint32_t*>(a.lo0);
  const uint32_t* lo1 = reinterpret_cast<const uint32_t*>(a.lo1);
  const uint32_t* hi0 = reinterpret_cast<const uint32_t*>(a.hi0);
  const uint32_t* hi1 = reinterpret_cast<const uint32_t*>(a.hi1);
  const uint32_t lane = threadIdx.x & 31u, S = kl.S;
  const uint64_t n = a.n, ngroups = (n + 7) >> 3;
  const uint64_t warps = (uint64_t)gridDim.x * (TPB / 32);
  for (uint64_t wb = ((uint64_t)blockIdx.x * (TPB / 32) + threadIdx.x / 32) * 256; wb < n; wb += warps * 256) {
    uint32_t zbits = 0;
#pragma unroll 1
    for (uint32_t e = 0; e < 8; ++e) {
      const uint64_t i = wb + 32 * e + lane;
      bool z = false;
      if (i < n) {  // step 9: any (W0_m + W1_m) mod p == 0
        const uint32_t h0 = hi0 ? __ldg(hi0 + i) : 0u, h1 = hi1 ? __ldg(hi1 + i) : 0u;
#pragma unroll 1
        for (uint32_t m0 = 0; m0 < S; m0 += 8) {
          uint32_t l0[8], l1[8];
#pragma unroll
          for (uint32_t k = 0; k < 8; ++k) {
            const bool ok = m0 + k < S;
            l0[k] = ok ? __ldg(lo0 + (m0 + k) * n + i) : 1u;  // absent slots: W0 + W1 = 2, never 0 or p
            l1[k] = ok ? __ldg(lo1 + (m0 + k) * n + i) : 1u;
          }
#pragma unroll
          for (uint32_t k = 0; k < 8; ++k) {
            const uint64_t W0 = (uint64_t)l0[k] | ((uint64_t)((h0 >> (m0 + k)) & 1u) << 32);
            const uint64_t W1 = (uint64_t)l1[k] | ((uint64_t)((h1 >> (m0 + k)) & 1u) << 32);
            const uint64_t sum = W0 + W1;
            z |= sum == 0 || sum == kl.p;
          }
        }
      }
      const uint32_t bal = __ballot_sync(0xFFFFFFFFu, z);  // elements wb + 32 e + 0..31
      if ((lane >> 2) == e) zbits = (bal >> (8 * (lane & 3u))) & 0xFFu;
    }
    const uint64_t g = wb / 8 + lane;
    if (g < ngroups) {
      const uint64_t i0 = g << 3;
      helper_respond<R, RELU, HI0>(a, kp, sp, i0, a.base + i0, (uint32_t)min((uint64_t)8, n - i0), zbits);
    }
  }
}

struct FinishArgs {
  const uint64_t* x;
  const uint8_t* tbits;
  const uint64_t* resp;  // DReLU: [D']_b (nullable for P0)    ReLU: e
  const uint64_t* d_own;
  const uint64_t* d_peer;
  const uint64_t* c1;
  uint64_t* y;
  uint64_t n, base;
};

template <int R, int PARTY, bool RELU, bool HI0 = false>
__global__ void __launch_bounds__(TPB, 2) k_finish(FinishArgs a, KP kp, const __grid_constant__ StreamPre sp) {
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB) {
    const uint64_t i0 = g << 3;
    const uint64_t j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    const uint32_t tb = a.tbits[g];
    uint64_t y[8];
    if (!RELU) {  // Alg 7 step 11
      uint64_t D[8];
      if (a.resp) {
        load8(a.resp + i0, D, cnt);
      } else {  // P0 derives [D']_0 from seed02 (reading C12)
        uint32_t Q[16];
        chacha_pre<R, HI0>(sp.resp, j0 >> 3, Q);
#pragma unroll
        for (int e = 0; e < 8; ++e) D[e] = u64_of(Q, e);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint64_t t = (tb >> e) & 1u, d = D[e] & kp.ymask;
        y[e] = PARTY == 0 ? (t ? (1ull - d) & kp.ymask : d) : (t ? (0ull - d) & kp.ymask : d);
      }
    } else {  // Alg 8 steps 4-5
      // [a]_b is not regenerated: the send phase published [d]_b = [x]_b - [a]_b, so
      // [a]_b = [x]_b - [d]_b (mod 2^ell) from the two vectors this phase reads anyway,
      // one ChaCha block per 8 elements fewer than drawing it again from the triple stream
      uint64_t x[8], ev[8], acc[8], own[8];
      load8(a.x + i0, x, cnt);
      load8(a.resp + i0, ev, cnt);
      {
        uint64_t dp[8];
        load8(a.d_own + i0, own, cnt);
        load8(a.d_peer + i0, dp, cnt);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = own[e] + dp[e];  // d = [d]_0 + [d]_1 (opened)
      }
      uint32_t Bk[16];
      chacha_pre<R, HI0>(PARTY == 0 ? sp.b02 : sp.b12, j0 >> 3, Bk);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint64_t d = acc[e], ab = x[e] - own[e];  // [a]_b
        acc[e] = d * u64_of(Bk, e) + ev[e] * ab + (PARTY == 0 ? d * ev[e] : 0ull);
      }
      if (PARTY == 0) {
        uint32_t Ck[16];
        chacha_pre<R, HI0>(sp.c02, j0 >> 3, Ck);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += u64_of(Ck, e);
      } else {
        uint64_t c1[8];
        load8(a.c1 + i0, c1, cnt);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += c1[e];
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint64_t t = (tb >> e) & 1u;
        y[e] = ((t ? x[e] : 0ull) + (t ? 0ull - acc[e] : acc[e])) & kp.ymask;
      }
    }
    store8(a.y + i0, y, cnt);
  }
}

template <bool RELU>
int send(int party, const uint64_t* x, uint8_t* lo, uint8_t* hi, uint8_t* tbits, uint64_t* dshare, uint64_t* dpeer,
         size_t n, uint64_t base, const bc_params* prm, const uint8_t* s01, const uint8_t* str, void* stream,
         uint64_t* y0 = nullptr) {
  const int rc = check_params(prm);
  if (rc) return rc;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if ((party != 0 && party != 1) || !x || !lo || (!tbits && !y0) || !s01 || (RELU && (!dshare || !str)))
    return BC_EINVAL;
  if (y0 && (RELU || party != 0 || !str)) return BC_EINVAL;  // P0's DReLU output needs seed02 (in str)
  if (y0 && !aligned16(y0)) return BC_EALIGN;
  const bool large = prm->tape == BC_TAPE_LARGE;
  if (!hi && prm->p > (large ? 0xFFFFFFFFull : 256ull)) return BC_EINVAL;  // the high-bit plane is needed
  if (!RELU && dpeer) return BC_EINVAL;
  if (!aligned16(x) || !aligned16(lo) || (hi && !aligned8(hi)) || (RELU && !aligned16(dshare)) ||
      (dpeer && !aligned16(dpeer)) || (base & 7))
    return BC_EALIGN;
  if (!index_range_ok(base, n)) return BC_ERANGE;  // global indices j < BC_MAX_INDEX
  const size_t nb = n * 8;
  const size_t nlo = large ? n * prm->slots * 4 : nb, nhi = large ? n * 4 : n;  // wire planes (bytes)
  if (overlap(lo, nlo, x, nb) || overlap(hi, nhi, x, nb) || overlap(tbits, (n + 7) / 8, x, nb) ||
      overlap(lo, nlo, hi, nhi) || overlap(lo, nlo, tbits, (n + 7) / 8) || overlap(hi, nhi, tbits, (n + 7) / 8) ||
      (RELU && (overlap(dshare, nb, x, nb) || overlap(dshare, nb, lo, nlo) || overlap(dshare, nb, hi, nhi))) ||
      overlap(dpeer, nb, x, nb) || overlap(dpeer, nb, dshare, nb) || overlap(y0, nb, x, nb) ||
      overlap(y0, nb, lo, nlo) || overlap(y0, nb, hi, nhi) || overlap(y0, nb, tbits, (n + 7) / 8))
    return BC_EALIAS;
  SendArgs a{x, lo, hi, tbits, dshare, dpeer, y0, (uint64_t)n, base};
  const KP kp = make_kp(prm);
  const Key k01 = make_key(s01);
  const Key ktr = (RELU || y0) ? make_key(str) : Key{};  // triple seed (ReLU) or seed02 (P0's DReLU output)
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t ngroups = (n + 7) / 8;
  return dispatch_rounds(prm->rounds, [&](auto Rc) {
    constexpr int R = decltype(Rc)::value;
    auto go = [&](auto fn) { fn<<<grid_for((const void*)fn, ngroups), TPB, 0, st>>>(a, kp, k01, ktr); };
    if (large) {
      const KPL kl = make_kpl(prm);
      const KeyPre tpl = make_keypre(s01, L_TAPEL);
      const bool c32 = base + n <= (1ull << 32) / 7;  // every tape counter 7j + b below 2^32
      auto pick = [&](auto P) {
        constexpr int PARTY = decltype(P)::value;
        if (kl.w == 31 && kl.S == 32 && kl.p == P31)  // the paper-literal full precision, p = 2^31 + 11
          return c32 ? k_send_l<R, PARTY, RELU, false, true, true> : k_send_l<R, PARTY, RELU, false, false, true>;
        return kl.w == 32 ? (c32 ? k_send_l<R, PARTY, RELU, true, true> : k_send_l<R, PARTY, RELU, true, false>)
                          : (c32 ? k_send_l<R, PARTY, RELU, false, true> : k_send_l<R, PARTY, RELU, false, false>);
      };
      auto fn = party == 0 ? pick(std::integral_constant<int, 0>{}) : pick(std::integral_constant<int, 1>{});
      fn<<<grid_for((const void*)fn, ngroups, TPB_LARGE), TPB_LARGE, 0, st>>>(a, kp, kl, k01, ktr, tpl);
    } else if (prm->tape == BC_TAPE_COMPACT && BC_SEND_TABLES) {
      SendPre sp{};
      sp.tpa = make_keypre(s01, L_TAPEA);
      sp.tpb = make_keypre(s01, L_TAPEB);
      if (RELU) sp.tra = make_keypre(str, party == 0 ? L_A02 : L_A12);
      if (!RELU && y0) sp.resp = make_keypre(str, L_RESP);
      const bool fhi = kp.fhi != 0, hi0 = base + n <= (1ull << 34);
      auto pick = [&](auto P) {
        constexpr int PARTY = decltype(P)::value;
        return fhi ? (hi0 ? k_send_t<R, PARTY, RELU, true, true> : k_send_t<R, PARTY, RELU, true, false>)
                   : (hi0 ? k_send_t<R, PARTY, RELU, false, true> : k_send_t<R, PARTY, RELU, false, false>);
      };
      auto fn = party == 0 ? pick(std::integral_constant<int, 0>{}) : pick(std::integral_constant<int, 1>{});
      const int rc = allow_smem((const void*)fn, kSendTabBytes);
      if (rc) return rc;
      fn<<<grid_for((const void*)fn, ngroups, TPB_ST, kSendTabBytes), TPB_ST, kSendTabBytes, st>>>(a, kp, k01, ktr, sp);
    } else if (prm->tape == BC_TAPE_COMPACT) {
      if (party == 0) go(k_send_c<R, 0, RELU>);
      else go(k_send_c<R, 1, RELU>);
    } else if (prm->tape == BC_TAPE_COMPACT_LIT) {
      if (party == 0) go(k_send_w<R, 0, RELU, true>);
      else go(k_send_w<R, 1, RELU, true>);
    } else {
      if (party == 0) go(k_send_w<R, 0, RELU, false>);
      else go(k_send_w<R, 1, RELU, false>);
    }
    return check_launch();
  });
}

template <bool RELU>
int helper(const uint8_t* lo0, const uint8_t* hi0, const uint8_t* lo1, const uint8_t* hi1, uint64_t* out0,
           uint64_t* out0b, uint64_t* out1, size_t n, uint64_t base, const bc_params* prm, const uint8_t* s02, const uint8_t* s12,
           void* stream) {
  const int rc = check_params(prm);
  if (rc) return rc;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if (!lo0 || !lo1 || !s02 || (RELU && (!s12 || !out0)) || (!RELU && !out1)) return BC_EINVAL;
  const bool large = prm->tape == BC_TAPE_LARGE;
  if (prm->p > (large ? 0xFFFFFFFFull : 256ull) && (!hi0 || !hi1)) return BC_EINVAL;
  if (!aligned16(lo0) || !aligned16(lo1) || (hi0 && !aligned8(hi0)) || (hi1 && !aligned8(hi1)) ||
      (out0 && !aligned16(out0)) || (out0b && !aligned16(out0b)) || (out1 && !aligned16(out1)) || (base & 7))
    return BC_EALIGN;
  if (!index_range_ok(base, n)) return BC_ERANGE;  // global indices j < BC_MAX_INDEX
  if (out0b && !out0) return BC_EINVAL;
  const size_t nb = n * 8;
  const size_t nlo = large ? n * prm->slots * 4 : nb, nhi = large ? n * 4 : n;  // wire planes (bytes)
  if (overlap(out0, nb, lo0, nlo) || overlap(out0, nb, lo1, nlo) || overlap(out1, nb, lo0, nlo) ||
      overlap(out1, nb, lo1, nlo) || overlap(out0, nb, out1, nb) || overlap(out0, nb, hi0, nhi) ||
      overlap(out0, nb, hi1, nhi) || overlap(out1, nb, hi0, nhi) || overlap(out1, nb, hi1, nhi) ||
      overlap(out0b, nb, out0, nb) || overlap(out0b, nb, out1, nb) || overlap(out0b, nb, lo0, nlo) ||
      overlap(out0b, nb, lo1, nlo) || overlap(out0b, nb, hi0, nhi) || overlap(out0b, nb, hi1, nhi))
    return BC_EALIAS;
  HelperArgs a{lo0, hi0, lo1, hi1, out0, out0b, out1, (uint64_t)n, base};
  const KP kp = make_kp(prm);
  StreamPre sp{};
  if (RELU) {
    sp.b02 = make_keypre(s02, L_B02);
    sp.a02 = make_keypre(s02, L_A02);
    sp.c02 = make_keypre(s02, L_C02);
    sp.b12 = make_keypre(s12, L_B12);
    sp.a12 = make_keypre(s12, L_A12);
  } else {
    sp.resp = make_keypre(s02, L_RESP);
  }
  const bool c32 = base + n <= (1ull << 35);  // every counter j / 8 below 2^32
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t ngroups = (n + 7) / 8;
  return dispatch_rounds(prm->rounds, [&](auto Rc) {
    constexpr int R = decltype(Rc)::value;
    if (large) {
      auto fn = c32 ? k_helper_l<R, RELU, true> : k_helper_l<R, RELU, false>;
      fn<<<grid_for((const void*)fn, ngroups), TPB, 0, st>>>(a, kp, make_kpl(prm), sp);
    } else {
      auto fn = c32 ? k_helper<R, RELU, true> : k_helper<R, RELU, false>;
      fn<<<grid_for((const void*)fn, ngroups), TPB, 0, st>>>(a, kp, sp);
    }
    return check_launch();
  });
}

template <bool RELU>
int finish(int party, const uint64_t* x, const uint8_t* tbits, const uint64_t* resp, const uint64_t* d_own,
           const uint64_t* d_peer, const uint64_t* c1, uint64_t* y, size_t n, uint64_t base, const bc_params* prm,
           const uint8_t* seed, void* stream) {
  const int rc = check_params(prm);
  if (rc) return rc;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if ((party != 0 && party != 1) || !tbits || !y) return BC_EINVAL;
  if (!RELU && !resp && (party != 0 || !seed)) return BC_EINVAL;
  if (RELU && (!x || !resp || !d_own || !d_peer || !seed || (party == 1 && !c1))) return BC_EINVAL;
  if (!aligned16(y) || (resp && !aligned16(resp)) || (x && !aligned16(x)) || (d_own && !aligned16(d_own)) ||
      (d_peer && !aligned16(d_peer)) || (c1 && !aligned16(c1)) || (base & 7))
    return BC_EALIGN;
  if (!index_range_ok(base, n)) return BC_ERANGE;  // global indices j < BC_MAX_INDEX
  const size_t nb = n * 8;
  if (overlap(y, nb, resp, nb) || overlap(y, nb, x, nb) || overlap(y, nb, d_own, nb) || overlap(y, nb, d_peer, nb) ||
      overlap(y, nb, c1, nb) || overlap(y, nb, tbits, (n + 7) / 8))
    return BC_EALIAS;
  FinishArgs a{x, tbits, resp, d_own, d_peer, party == 1 ? c1 : nullptr, y, (uint64_t)n, base};
  const KP kp = make_kp(prm);
  StreamPre sp{};  // the finishing party's own seed: seed02 (P0) or seed12 (P1)
  if (seed) {
    if (!RELU) {
      sp.resp = make_keypre(seed, L_RESP);
    } else if (party == 0) {
      sp.b02 = make_keypre(seed, L_B02);
      sp.c02 = make_keypre(seed, L_C02);
    } else {
      sp.b12 = make_keypre(seed, L_B12);
    }
  }
  const bool hi0 = base + n <= (1ull << 35);  // every counter j / 8 below 2^32
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t ngroups = (n + 7) / 8;
  return dispatch_rounds(prm->rounds, [&](auto Rc) {
    constexpr int R = decltype(Rc)::value;
    auto go = [&](auto fn) { fn<<<grid_for((const void*)fn, ngroups), TPB, 0, st>>>(a, kp, sp); };
    if (party == 0) hi0 ? go(k_finish<R, 0, RELU, true>) : go(k_finish<R, 0, RELU, false>);
    else hi0 ? go(k_finish<R, 1, RELU, true>) : go(k_finish<R, 1, RELU, false>);
    return check_launch();
  });
}

}  // namespace

extern "C" {

int bc_drelu_send(int party, const uint64_t* x, uint8_t* lo, uint8_t* hi, uint8_t* tbits, size_t n,
                  uint64_t elem_base, const bc_params* prm, const uint8_t seed01[32], void* stream) {
  return send<false>(party, x, lo, hi, tbits, nullptr, nullptr, n, elem_base, prm, seed01, nullptr, stream);
}

int bc_drelu_send_p0(const uint64_t* x, uint8_t* lo, uint8_t* hi, uint8_t* tbits, uint64_t* y, size_t n,
                     uint64_t elem_base, const bc_params* prm, const uint8_t seed01[32], const uint8_t seed02[32],
                     void* stream) {
  if (!y) return BC_EINVAL;
  return send<false>(0, x, lo, hi, tbits, nullptr, nullptr, n, elem_base, prm, seed01, seed02, stream, y);
}

int bc_drelu_helper(const uint8_t* lo0, const uint8_t* hi0, const uint8_t* lo1, const uint8_t* hi1, uint64_t* resp0,
                    uint64_t* resp1, size_t n, uint64_t elem_base, const bc_params* prm, const uint8_t seed02[32],
                    void* stream) {
  return helper<false>(lo0, hi0, lo1, hi1, resp0, nullptr, resp1, n, elem_base, prm, seed02, nullptr, stream);
}

int bc_drelu_finish(int party, const uint8_t* tbits, const uint64_t* resp, uint64_t* y, size_t n, uint64_t elem_base,
                    const bc_params* prm, const uint8_t seed02[32], void* stream) {
  return finish<false>(party, nullptr, tbits, resp, nullptr, nullptr, nullptr, y, n, elem_base, prm, seed02, stream);
}

int bc_relu_send(int party, const uint64_t* x, uint8_t* lo, uint8_t* hi, uint8_t* tbits, uint64_t* dshare, size_t n,
                 uint64_t elem_base, const bc_params* prm, const uint8_t seed01[32], const uint8_t seed_tr[32],
                 void* stream) {
  return send<true>(party, x, lo, hi, tbits, dshare, nullptr, n, elem_base, prm, seed01, seed_tr, stream);
}

int bc_relu_send_to(int party, const uint64_t* x, uint8_t* lo, uint8_t* hi, uint8_t* tbits, uint64_t* dshare,
                    uint64_t* dshare_peer, size_t n, uint64_t elem_base, const bc_params* prm,
                    const uint8_t seed01[32], const uint8_t seed_tr[32], void* stream) {
  return send<true>(party, x, lo, hi, tbits, dshare, dshare_peer, n, elem_base, prm, seed01, seed_tr, stream);
}

int bc_relu_helper(const uint8_t* lo0, const uint8_t* hi0, const uint8_t* lo1, const uint8_t* hi1, uint64_t* e,
                   uint64_t* c1, size_t n, uint64_t elem_base, const bc_params* prm, const uint8_t seed02[32],
                   const uint8_t seed12[32], void* stream) {
  return helper<true>(lo0, hi0, lo1, hi1, e, nullptr, c1, n, elem_base, prm, seed02, seed12, stream);
}

int bc_relu_helper_to(const uint8_t* lo0, const uint8_t* hi0, const uint8_t* lo1, const uint8_t* hi1, uint64_t* e0,
                      uint64_t* e1, uint64_t* c1, size_t n, uint64_t elem_base, const bc_params* prm,
                      const uint8_t seed02[32], const uint8_t seed12[32], void* stream) {
  return helper<true>(lo0, hi0, lo1, hi1, e0, e1, c1, n, elem_base, prm, seed02, seed12, stream);
}

int bc_relu_finish(int party, const uint64_t* x, const uint8_t* tbits, const uint64_t* d_own, const uint64_t* d_peer,
                   const uint64_t* e, const uint64_t* c1, uint64_t* y, size_t n, uint64_t elem_base,
                   const bc_params* prm, const uint8_t seed_tr[32], void* stream) {
  return finish<true>(party, x, tbits, e, d_own, d_peer, c1, y, n, elem_base, prm, seed_tr, stream);
}

}  // extern "C"
