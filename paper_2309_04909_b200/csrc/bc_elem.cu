// bc_elem.cu -- elementwise primitives, HBM-bound: Alg 4/5 deterministic
// truncation, Alg 1 SecureML truncation, Alg 6 modulo switch and Alg 7 steps
// 3-5 (ladder + pairwise + modulo switch).  Two elements per thread per
// iteration: one 16-B load and one 16-B (or 8-B) store, fully coalesced.
#include "bc_common.cuh"

using namespace bc;
using namespace bc::host;

namespace {

struct EwArgs {
  const uint64_t* in;
  void* out;
  uint64_t n;
  uint64_t ymask;   // output modulus mask
  uint64_t inmask;  // 2^ell - 1
  uint32_t k1;
  uint32_t lp, p;
  int party;
};

__device__ __forceinline__ void load_pair(const uint64_t* __restrict__ in, uint64_t i, uint64_t n, uint64_t (&v)[2]) {
  if (2 * i + 1 < n) {
    const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(in) + i);
    v[0] = t.x;
    v[1] = t.y;
  } else {
    v[0] = __ldg(in + 2 * i);
    v[1] = 0;
  }
}

__device__ __forceinline__ void store_pair(uint64_t* __restrict__ out, uint64_t i, uint64_t n, const uint64_t (&v)[2]) {
  if (2 * i + 1 < n) reinterpret_cast<ulonglong2*>(out)[i] = make_ulonglong2(v[0], v[1]);
  else out[2 * i] = v[0];
}

// Alg 5 (k2 = 0: Alg 4): P0 cut(x, k1, k2); P1 -cut(-x, k1, k2), mod 2^(ell-k1-k2).
__global__ void __launch_bounds__(TPB) k_trc(EwArgs a) {
  const uint64_t npairs = (a.n + 1) >> 1;
  for (uint64_t i = (uint64_t)blockIdx.x * TPB + threadIdx.x; i < npairs; i += (uint64_t)gridDim.x * TPB) {
    uint64_t v[2];
    load_pair(a.in, i, a.n, v);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint64_t x = a.party == 0 ? v[k] : (0ull - v[k]) & a.inmask;
      const uint64_t c = (x >> a.k1) & a.ymask;
      v[k] = a.party == 0 ? c : (0ull - c) & a.ymask;
    }
    store_pair(static_cast<uint64_t*>(a.out), i, a.n, v);
  }
}

// Alg 1: P0 cut(x, k) mod 2^ell; P1 2^ell - cut(2^ell - x, k) mod 2^ell (reading C3).
__global__ void __launch_bounds__(TPB) k_trc_prob(EwArgs a) {
  const uint64_t npairs = (a.n + 1) >> 1;
  for (uint64_t i = (uint64_t)blockIdx.x * TPB + threadIdx.x; i < npairs; i += (uint64_t)gridDim.x * TPB) {
    uint64_t v[2];
    load_pair(a.in, i, a.n, v);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint64_t x = v[k] & a.inmask;
      v[k] = a.party == 0 ? (x >> a.k1) : (0ull - (((0ull - x) & a.inmask) >> a.k1)) & a.inmask;
    }
    store_pair(static_cast<uint64_t*>(a.out), i, a.n, v);
  }
}

// Alg 6.
__global__ void __launch_bounds__(TPB) k_modswitch(EwArgs a) {
  const uint64_t npairs = (a.n + 1) >> 1;
  const uint64_t lmask = (1ull << a.lp) - 1ull;
  const uint64_t two_lp = 1ull << a.lp;
  uint32_t* out = static_cast<uint32_t*>(a.out);
  const bool vec = (reinterpret_cast<uintptr_t>(out) & 7) == 0;
  for (uint64_t i = (uint64_t)blockIdx.x * TPB + threadIdx.x; i < npairs; i += (uint64_t)gridDim.x * TPB) {
    uint64_t v[2];
    load_pair(a.in, i, a.n, v);
    uint32_t o[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint64_t x = v[k] & lmask;
      if (a.party == 0) o[k] = (uint32_t)(x == 0 ? two_lp % a.p : x % a.p);
      else o[k] = (uint32_t)(((uint64_t)a.p + x - two_lp) % a.p);
    }
    if (2 * i + 1 < a.n && vec) {
      reinterpret_cast<uint2*>(out)[i] = make_uint2(o[0], o[1]);
    } else {
      out[2 * i] = o[0];
      if (2 * i + 1 < a.n) out[2 * i + 1] = o[1];
    }
  }
}

// Alg 7 steps 3-5 on the share as given: bytes v'_m - 1 (slot m -> byte m).
template <int PARTY>
__device__ __forceinline__ uint64_t ladder_bytes(uint64_t x, const KP& kp, bool compact) {
  const uint32_t win = window_of<PARTY>(x, 0u, kp.fsh, kp.fhi != 0);  // P1 works on -[x]_1 (reading C3)
  if (compact) {  // w = 8, p = 257: all 8 windows at once (SWAR)
    uint32_t lo, hi;
    ladder_swar<PARTY>(win, lo, hi);
    return (uint64_t)lo | ((uint64_t)hi << 32);
  }
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t b = (win >> i) & kp.wmask;
    u[i] = PARTY == 0 ? b : ((0u - b) & kp.wmask);
  }
  uint64_t out = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if ((uint32_t)i <= kp.lx) {
      const uint32_t nxt = ((uint32_t)i < kp.lx) ? u[i + 1] : 0u;
      const uint32_t vi = (u[i] + nxt - (PARTY == 0 ? 1u : 0u)) & kp.wmask;
      uint32_t vp;
      if (PARTY == 0) vp = (vi == 0) ? modp_small(1u << kp.w, kp) : modp_small(vi, kp);
      else vp = modp_small(kp.p + vi - (1u << kp.w), kp);
      out |= (uint64_t)(vp - 1u) << (8 * i);
    }
  }
  return out;
}

#ifndef BC_LADDER_ILP
#define BC_LADDER_ILP 2  // measured at 2^28: 1: 0.711-0.713 ms, 2: 0.704 (6,102 GB/s), 4: 0.748
#endif
#ifndef BC_LADDER_CS
#define BC_LADDER_CS 0  // 1: streaming (evict-first) loads and stores; measured: no gain (0.712 / 0.705 with ILP 2)
#endif
__device__ __forceinline__ void load_pair_cs(const uint64_t* __restrict__ in, uint64_t i, uint64_t n, uint64_t (&v)[2]) {
  if (!BC_LADDER_CS) return load_pair(in, i, n, v);
  if (2 * i + 1 < n) {
    const ulonglong2 t = __ldcs(reinterpret_cast<const ulonglong2*>(in) + i);
    v[0] = t.x;
    v[1] = t.y;
  } else {
    v[0] = __ldcs(in + 2 * i);
    v[1] = 0;
  }
}
__device__ __forceinline__ void store_pair_cs(uint64_t* __restrict__ out, uint64_t i, uint64_t n, const uint64_t (&v)[2]) {
  if (!BC_LADDER_CS) return store_pair(out, i, n, v);
  if (2 * i + 1 < n) __stcs(reinterpret_cast<ulonglong2*>(out) + i, make_ulonglong2(v[0], v[1]));
  else __stcs(out + 2 * i, v[0]);
}
template <int PARTY>
__global__ void __launch_bounds__(TPB) k_ladder(const uint64_t* __restrict__ x, uint64_t* __restrict__ v, uint64_t n,
                                                KP kp, int compact) {
  const uint64_t npairs = (n + 1) >> 1;
  const uint64_t stride = (uint64_t)gridDim.x * TPB;
  // BC_LADDER_ILP pairs per iteration, their loads issued before any compute (more bytes in flight)
  for (uint64_t i = (uint64_t)blockIdx.x * TPB + threadIdx.x; i < npairs; i += BC_LADDER_ILP * stride) {
    uint64_t t[BC_LADDER_ILP][2];
#pragma unroll
    for (int k = 0; k < BC_LADDER_ILP; ++k)
      if (k == 0 || i + k * stride < npairs) load_pair_cs(x, i + k * stride, n, t[k]);
#pragma unroll
    for (int k = 0; k < BC_LADDER_ILP; ++k) {
      if (k == 0 || i + k * stride < npairs) {
        t[k][0] = ladder_bytes<PARTY>(t[k][0], kp, compact);
        t[k][1] = ladder_bytes<PARTY>(t[k][1], kp, compact);
        store_pair_cs(v, i + k * stride, n, t[k]);
      }
    }
  }
}

// Alg 6 at any width: 1 <= lp <= 63, 2^lp < p < 2^64.  Both results are
// already reduced: P0's x < 2^lp < p (and 2^lp mod p = 2^lp), P1's p - 2^lp + x < p.
__global__ void __launch_bounds__(TPB) k_modswitch64(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                     uint64_t n, uint32_t lp, uint64_t p, int party) {
  const uint64_t npairs = (n + 1) >> 1;
  const uint64_t two_lp = 1ull << lp, lmask = two_lp - 1ull;
  for (uint64_t i = (uint64_t)blockIdx.x * TPB + threadIdx.x; i < npairs; i += (uint64_t)gridDim.x * TPB) {
    uint64_t v[2];
    load_pair(in, i, n, v);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint64_t x = v[k] & lmask;
      v[k] = party == 0 ? (x == 0 ? two_lp : x) : (p - two_lp) + x;
    }
    store_pair(out, i, n, v);
  }
}

// Alg 7 steps 3-5 for one party, any tape (up to 32 slots, p < 2^33): v'_m as uint64_t[n][S].
// A warp owns 32 consecutive elements; element e's row is written by lanes m < S together
// (S consecutive words), lane m computing slot m from the broadcast share.
struct Lad64 {
  const uint64_t* x;
  uint64_t* v;
  uint64_t n, inmask, wmask, two_w, p;
  uint32_t f, lx, S;
};
template <int PARTY>
__global__ void __launch_bounds__(TPB) k_ladder64(Lad64 a) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t nwarps = (uint64_t)gridDim.x * (TPB / 32);
  for (uint64_t wbase = ((uint64_t)blockIdx.x * (TPB / 32) + threadIdx.x / 32) * 32; wbase < a.n;
       wbase += nwarps * 32) {
    const uint64_t i = wbase + lane;
    const uint64_t xi = i < a.n ? __ldg(a.x + i) : 0ull;
    const uint32_t cnt = (uint32_t)min((uint64_t)32, a.n - wbase);
    for (uint32_t e = 0; e < cnt; ++e) {
      const uint64_t s = __shfl_sync(0xFFFFFFFFu, xi, (int)e);
      if (lane >= a.S) continue;
      // Alg 5 windows (k1 = f + m): P0 reads s, P1 reads -s (reading C3) and negates the window (C4)
      const uint64_t op = PARTY == 0 ? (s & a.inmask) : ((0ull - s) & a.inmask);
      uint64_t u = (op >> (a.f + lane)) & a.wmask;
      uint64_t u1 = lane < a.lx ? (op >> (a.f + lane + 1)) & a.wmask : 0ull;
      if (PARTY == 1) { u = (0ull - u) & a.wmask; u1 = (0ull - u1) & a.wmask; }
      const uint64_t vm = (u + u1 - (PARTY == 0 ? 1ull : 0ull)) & a.wmask;  // P0 carries the -1 (C8)
      // Alg 6: P0 v = 0 -> 2^w (= 2^w mod p); P1 p + v - 2^w (both already in [1, p))
      a.v[(wbase + e) * a.S + lane] = PARTY == 0 ? (vm == 0 ? a.two_w : vm) : (a.p - a.two_w) + vm;
    }
  }
}

}  // namespace

extern "C" {

int bc_modswitch64(int party, const uint64_t* in, uint64_t* out, size_t n, int lp, uint64_t p, void* stream) {
  if ((party != 0 && party != 1) || lp < 1 || lp > 63 || p <= (1ull << lp)) return BC_EINVAL;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if (!in || !out) return BC_EINVAL;
  if (!aligned16(in) || !aligned16(out)) return BC_EALIGN;
  if (overlap(in, n * 8, out, n * 8)) return BC_EALIAS;
  k_modswitch64<<<grid_for((const void*)k_modswitch64, (n + 1) / 2), TPB, 0, static_cast<cudaStream_t>(stream)>>>(
      in, out, n, (uint32_t)lp, p, party);
  return check_launch();
}

int bc_ladder_modswitch64(int party, const uint64_t* x, uint64_t* v, size_t n, const bc_params* prm, void* stream) {
  const int rc = check_params(prm);
  if (rc) return rc;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if (party != 0 && party != 1) return BC_EINVAL;
  if (!x || !v) return BC_EINVAL;
  if (!aligned16(x) || !aligned16(v)) return BC_EALIGN;
  if (overlap(x, n * 8, v, n * 8 * prm->slots)) return BC_EALIAS;
  Lad64 a{};
  a.x = x;
  a.v = v;
  a.n = n;
  a.inmask = prm->ell == 64 ? ~0ull : ((1ull << prm->ell) - 1ull);
  a.two_w = 1ull << prm->w;
  a.wmask = a.two_w - 1ull;
  a.p = prm->p;
  a.f = (uint32_t)prm->f;
  a.lx = (uint32_t)prm->lx;
  a.S = prm->slots;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t warps = (n + 31) / 32;
  if (party == 0)
    k_ladder64<0><<<grid_for((const void*)k_ladder64<0>, warps * 32), TPB, 0, st>>>(a);
  else
    k_ladder64<1><<<grid_for((const void*)k_ladder64<1>, warps * 32), TPB, 0, st>>>(a);
  return check_launch();
}

int bc_trc(int party, const uint64_t* in, uint64_t* out, size_t n, int ell, int k1, int k2, void* stream) {
  if ((party != 0 && party != 1) || ell < 2 || ell > 64 || k1 < 0 || k2 < 0 || k1 + k2 >= ell)
    return BC_EINVAL;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if (!in || !out) return BC_EINVAL;
  if (!aligned16(in) || !aligned16(out)) return BC_EALIGN;
  if (overlap(in, n * 8, out, n * 8)) return BC_EALIAS;
  const int lp = ell - k1 - k2;
  EwArgs a{};
  a.in = in;
  a.out = out;
  a.n = n;
  a.party = party;
  a.k1 = (uint32_t)k1;
  a.ymask = lp == 64 ? ~0ull : ((1ull << lp) - 1ull);
  a.inmask = ell == 64 ? ~0ull : ((1ull << ell) - 1ull);
  k_trc<<<grid_for((const void*)k_trc, (n + 1) / 2), TPB, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return check_launch();
}

int bc_trc_prob(int party, const uint64_t* in, uint64_t* out, size_t n, int ell, int k, void* stream) {
  if ((party != 0 && party != 1) || ell < 2 || ell > 64 || k < 0 || k >= ell) return BC_EINVAL;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if (!in || !out) return BC_EINVAL;
  if (!aligned16(in) || !aligned16(out)) return BC_EALIGN;
  if (overlap(in, n * 8, out, n * 8)) return BC_EALIAS;
  EwArgs a{};
  a.in = in;
  a.out = out;
  a.n = n;
  a.party = party;
  a.k1 = (uint32_t)k;
  a.inmask = ell == 64 ? ~0ull : ((1ull << ell) - 1ull);
  k_trc_prob<<<grid_for((const void*)k_trc_prob, (n + 1) / 2), TPB, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return check_launch();
}

int bc_modswitch(int party, const uint64_t* in, uint32_t* out, size_t n, int lp, uint32_t p, void* stream) {
  if ((party != 0 && party != 1) || lp < 1 || lp > 31 || (uint64_t)p <= (1ull << lp))
    return BC_EINVAL;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if (!in || !out) return BC_EINVAL;
  if (!aligned16(in) || (reinterpret_cast<uintptr_t>(out) & 3)) return BC_EALIGN;
  if (overlap(in, n * 8, out, n * 4)) return BC_EALIAS;
  EwArgs a{};
  a.in = in;
  a.out = out;
  a.n = n;
  a.party = party;
  a.lp = (uint32_t)lp;
  a.p = p;
  k_modswitch<<<grid_for((const void*)k_modswitch, (n + 1) / 2), TPB, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return check_launch();
}

int bc_ladder_modswitch(int party, const uint64_t* x, uint8_t* v, size_t n, const bc_params* prm, void* stream) {
  const int rc = check_params(prm);
  if (rc) return rc;
  if (n == 0) return BC_OK;  // no-op after parameter validation
  if (party != 0 && party != 1) return BC_EINVAL;
  if (prm->tape == BC_TAPE_LARGE) return BC_EINVAL;  // byte format: slots <= 8, p <= 257
  if (!aligned16(x) || !aligned16(v)) return BC_EALIGN;
  if (overlap(x, n * 8, v, n * 8)) return BC_EALIAS;
  const KP kp = make_kp(prm);
  const int compact = prm->tape == BC_TAPE_COMPACT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t* vo = reinterpret_cast<uint64_t*>(v);
  if (party == 0)
    k_ladder<0><<<grid_for((const void*)k_ladder<0>, (n + 1) / 2), TPB, 0, st>>>(x, vo, n, kp, compact);
  else
    k_ladder<1><<<grid_for((const void*)k_ladder<1>, (n + 1) / 2), TPB, 0, st>>>(x, vo, n, kp, compact);
  return check_launch();
}

}  // extern "C"
