// bc_trunc.cu -- the truncation study: Alg 2 (ABY3,
// P:329-342) fused for both parties, exact e1 counting over mask ranges
// (sec. 4; classes of reading C30), and Alg 3 truncate-then-multiply
// against multiply-then-truncate (sec. 5.2) with a seed-derived
// Beaver triple (reading C31).
//
// Thread mapping as elsewhere: one thread owns 8 consecutive elements, so each
// 8-B-per-element stream is exactly one ChaCha block per thread.
#include "bc_common.cuh"

using namespace bc;
using namespace bc::host;

namespace {

constexpr int TPB_T = 128;

constexpr uint64_t L_T0R0 = lbl("bc2.t0r0"), L_T0R1 = lbl("bc2.t0r1"), L_T0Q0 = lbl("bc2.t0q0");
constexpr uint64_t L_T1R0 = lbl("bc2.t1r0"), L_T1R1 = lbl("bc2.t1r1"), L_T1Q0 = lbl("bc2.t1q0");
constexpr uint64_t L_MA02 = lbl("bc2.ma02"), L_MB02 = lbl("bc2.mb02"), L_MC02 = lbl("bc2.mc02");
constexpr uint64_t L_MA12 = lbl("bc2.ma12"), L_MB12 = lbl("bc2.mb12");

struct TP {
  uint64_t ymask;  // 2^ell - 1
  uint32_t ell;
};

template <int R>
__device__ __forceinline__ void stream8(const Key& k, uint64_t blk, uint64_t label, uint64_t (&v)[8]) {
  uint32_t B[16];
  chacha<R>(k, blk, label, B);
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = u64_of(B, e);
}

__device__ __forceinline__ void load8(const uint64_t* p, uint64_t i0, uint64_t n, uint64_t (&v)[8]) {
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const ulonglong2 u = load2(p, i0 + 2 * h, n);
    v[2 * h] = u.x;
    v[2 * h + 1] = u.y;
  }
}

// Alg 1 on 8 elements in place: P0 cut([x]_0, k), P1 -cut(-[x]_1, k).
__device__ __forceinline__ void secureml8(uint64_t (&a0)[8], uint64_t (&a1)[8], uint32_t k, const TP& tp) {
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    a0[e] = (a0[e] & tp.ymask) >> k;
    a1[e] = (0ull - (((0ull - a1[e]) & tp.ymask) >> k)) & tp.ymask;
  }
}

// Alg 2 (reading C29) on 8 elements in place, truncation instance q.
template <int R>
__device__ __forceinline__ void aby3_8(uint64_t (&a0)[8], uint64_t (&a1)[8], uint32_t k, const TP& tp,
                                       const Key& k02, const Key& k12, uint64_t blk, int q) {
  uint64_t r[8], t[8];
  stream8<R>(k02, blk, q ? L_T1R0 : L_T0R0, r);        // [r]_0 (P0, P2)
#pragma unroll
  for (int e = 0; e < 8; ++e) a0[e] += r[e];           // P0 publishes [x]_0 + [r]_0
  stream8<R>(k12, blk, q ? L_T1R1 : L_T0R1, t);        // [r]_1 (P1, P2)
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    a1[e] += t[e];                                     // P1 publishes [x]_1 + [r]_1
    r[e] = (r[e] + t[e]) & tp.ymask;                   // P2 (dealer) knows r
  }
  stream8<R>(k02, blk, q ? L_T1Q0 : L_T0Q0, t);        // [r']_0
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint64_t alpha = (a0[e] + a1[e]) & tp.ymask;  // step 1: alpha = x + r
    const uint64_t rp1 = (r[e] >> k) - t[e];           // P2 -> P1: [r']_1 = cut(r, k) - [r']_0
    a0[e] = ((alpha >> k) - t[e]) & tp.ymask;          // step 2, P0: alpha/2^k - [r']_0
    a1[e] = (0ull - rp1) & tp.ymask;                   //         P1: -[r']_1
  }
}

template <int R>
__device__ __forceinline__ void trc8(int alg, uint64_t (&a0)[8], uint64_t (&a1)[8], uint32_t k, const TP& tp,
                                     const Key& k02, const Key& k12, uint64_t blk, int q) {
  if (alg == BC_TRC_ABY3) aby3_8<R>(a0, a1, k, tp, k02, k12, blk, q);
  else secureml8(a0, a1, k, tp);
}

// Two-party Beaver product (reading C31): z_0 = de + d[b]_0 + e[a]_0 + [c]_0,
// z_1 = d[b]_1 + e[a]_1 + [c]_1 with [c]_1 = ab - [c]_0 from P2.
template <int R>
__device__ __forceinline__ void beaver8(uint64_t (&x0)[8], uint64_t (&x1)[8], const uint64_t (&y0)[8],
                                        const uint64_t (&y1)[8], const Key& k02, const Key& k12, uint64_t blk) {
  uint64_t a0[8], a1[8], b0[8], b1[8];
  stream8<R>(k02, blk, L_MA02, a0);
  stream8<R>(k12, blk, L_MA12, a1);
  stream8<R>(k02, blk, L_MB02, b0);
  stream8<R>(k12, blk, L_MB12, b1);
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint64_t d = (x0[e] - a0[e]) + (x1[e] - a1[e]);  // opened d = x - a
    const uint64_t ev = (y0[e] - b0[e]) + (y1[e] - b1[e]); // opened e = y - b
    x0[e] = d * ev + d * b0[e] + ev * a0[e];
    x1[e] = d * b1[e] + ev * a1[e] + (a0[e] + a1[e]) * (b0[e] + b1[e]);
  }
  stream8<R>(k02, blk, L_MC02, a0);                        // [c]_0
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    x0[e] += a0[e];
    x1[e] -= a0[e];
  }
}

struct TrcArgs {
  const uint64_t *x0, *x1;
  uint64_t *y0, *y1;
  uint64_t n, base;
};

template <int R>
__global__ void __launch_bounds__(TPB_T) k_trc_aby3(TrcArgs a, TP tp, uint32_t k, int q, Key k02, Key k12) {
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB_T + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB_T) {
    const uint64_t i0 = g << 3, j0 = a.base + i0;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint64_t s0[8], s1[8];
    load8(a.x0, i0, a.n, s0);
    load8(a.x1, i0, a.n, s1);
    aby3_8<R>(s0, s1, k, tp, k02, k12, j0 >> 3, q);
    store8(a.y0 + i0, s0, cnt);
    store8(a.y1 + i0, s1, cnt);
  }
}

struct MulArgs {
  const uint64_t *x0, *x1, *y0, *y1;
  uint64_t *z0, *z1;
  uint64_t n, base;
};

template <int R>
__global__ void __launch_bounds__(TPB_T) k_mul_trc(MulArgs a, TP tp, int order, int alg, uint32_t f, Key k02,
                                                   Key k12) {
  const uint64_t ngroups = (a.n + 7) >> 3;
  for (uint64_t g = (uint64_t)blockIdx.x * TPB_T + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * TPB_T) {
    const uint64_t i0 = g << 3, j0 = a.base + i0, blk = j0 >> 3;
    const uint32_t cnt = (uint32_t)min((uint64_t)8, a.n - i0);
    uint64_t u0[8], u1[8], v0[8], v1[8];
    load8(a.x0, i0, a.n, u0);
    load8(a.x1, i0, a.n, u1);
    load8(a.y0, i0, a.n, v0);
    load8(a.y1, i0, a.n, v1);
    if (order == BC_TRC_THEN_MUL) {                    // Alg 3: floor(f/2) bits of x, ceil(f/2) of y (C31)
      trc8<R>(alg, u0, u1, f / 2, tp, k02, k12, blk, 0);
      trc8<R>(alg, v0, v1, f - f / 2, tp, k02, k12, blk, 1);
      beaver8<R>(u0, u1, v0, v1, k02, k12, blk);
    } else {                                           // multiply, then truncate the product by f
      beaver8<R>(u0, u1, v0, v1, k02, k12, blk);
      trc8<R>(alg, u0, u1, f, tp, k02, k12, blk, 0);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      u0[e] &= tp.ymask;
      u1[e] &= tp.ymask;
    }
    store8(a.z0 + i0, u0, cnt);
    store8(a.z1 + i0, u1, cnt);
  }
}

// Exact e1 counting: CTA (i, c) runs x[i] against masks [m_base + c*CH, ...).
constexpr int CNT_TPB = 256;
constexpr uint64_t CNT_PER_THREAD = 64;
constexpr uint64_t CNT_CH = CNT_TPB * CNT_PER_THREAD;

__global__ void __launch_bounds__(CNT_TPB) k_trc_count(int alg, const uint64_t* __restrict__ xs, uint64_t nx,
                                                       uint32_t ell, uint32_t k, uint64_t m_base, uint64_t m_count,
                                                       uint64_t nchunks, unsigned long long* counts) {
  const uint64_t ymask = ell == 64 ? ~0ull : ((1ull << ell) - 1ull);
  const uint64_t omask = alg == BC_TRC_DET ? ((1ull << (ell - k)) - 1ull) : ymask;  // Alg 4 lives in Z_{2^(ell-k)}
  unsigned long long cnt[3] = {0, 0, 0};
  for (uint64_t b = blockIdx.x; b < nx * nchunks; b += gridDim.x) {
    const uint64_t i = b % nx, c = b / nx;
    const uint64_t x = __ldg(xs + i) & ymask;
    const bool pos = x < (1ull << (ell - 1));
    const uint64_t xi = pos ? x : (0ull - x) & ymask;
    const uint64_t cx = (xi >> k) & omask;
    const uint64_t T = pos ? cx : (0ull - cx) & omask;  // the expected trc (C30)
    const uint64_t one = pos ? 1ull : omask;            // the direction of the one-bit error
    const uint64_t lo = c * CNT_CH + threadIdx.x;
    for (uint64_t t = lo; t < min(m_count, (c + 1) * CNT_CH); t += CNT_TPB) {
      const uint64_t m = (m_base + t) & ymask;
      uint64_t y;
      if (alg == BC_TRC_ABY3) {                        // r = m; the x shares are (x, 0), the r' shares (cut(r,k), 0)
        const uint64_t alpha = (x + m) & ymask;
        y = ((alpha >> k) - (m >> k)) & ymask;
      } else {                                         // [x]_0 = x + m, [x]_1 = -m
        const uint64_t x0 = (x + m) & ymask, x1 = (0ull - m) & ymask;
        const uint64_t p0 = x0 >> k, p1 = ((0ull - x1) & ymask) >> k;
        y = alg == BC_TRC_DET ? (p0 - p1) & omask            // Alg 4: cut mod 2^(ell-k)
                              : ((p0 & ymask) + ((0ull - p1) & ymask)) & ymask;  // Alg 1
      }
      const uint64_t d = (y - T) & omask;
      cnt[d == 0 ? 0 : (d == one ? 1 : 2)] += 1;
    }
    // one atomic per warp and class
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      unsigned long long v = cnt[q];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
      if ((threadIdx.x & 31) == 0 && v) atomicAdd(counts + 3 * i + q, v);
      cnt[q] = 0;
    }
  }
}

bool valid_alg(int alg, bool det_ok) {
  return alg == BC_TRC_SECUREML || alg == BC_TRC_ABY3 || (det_ok && alg == BC_TRC_DET);
}

}  // namespace

extern "C" {

int bc_trc_aby3(const uint64_t* x0, const uint64_t* x1, uint64_t* y0, uint64_t* y1, size_t n, uint64_t elem_base,
                int ell, int k, int rounds, int q, const bc_seeds* seeds, void* stream) {
  if (ell < 2 || ell > 64 || k < 0 || k >= ell || (q != 0 && q != 1) || (rounds != 8 && rounds != 12 && rounds != 20))
    return BC_EINVAL;
  if (n == 0) return BC_OK;
  if (!x0 || !x1 || !y0 || !y1 || !seeds) return BC_EINVAL;
  if (!aligned16(x0) || !aligned16(x1) || !aligned16(y0) || !aligned16(y1) || (elem_base & 7)) return BC_EALIGN;
  if (!index_range_ok(elem_base, n)) return BC_ERANGE;  // global indices j < BC_MAX_INDEX
  const size_t nb = n * 8;
  if (overlap(y0, nb, y1, nb) || overlap(y0, nb, x0, nb) || overlap(y0, nb, x1, nb) || overlap(y1, nb, x0, nb) ||
      overlap(y1, nb, x1, nb))
    return BC_EALIAS;
  const TP tp{ell == 64 ? ~0ull : ((1ull << ell) - 1ull), (uint32_t)ell};
  const Key k02 = make_key(seeds->s02), k12 = make_key(seeds->s12);
  TrcArgs a{x0, x1, y0, y1, (uint64_t)n, elem_base};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return dispatch_rounds(rounds, [&](auto Rc) {
    constexpr int R = decltype(Rc)::value;
    auto fn = k_trc_aby3<R>;
    fn<<<grid_for((const void*)fn, (n + 7) / 8, TPB_T), TPB_T, 0, st>>>(a, tp, (uint32_t)k, q, k02, k12);
    return check_launch();
  });
}

int bc_mul_trc(int order, int alg, const uint64_t* x0, const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
               uint64_t* z0, uint64_t* z1, size_t n, uint64_t elem_base, int ell, int f, int rounds,
               const bc_seeds* seeds, void* stream) {
  if ((order != BC_MUL_THEN_TRC && order != BC_TRC_THEN_MUL) || !valid_alg(alg, false) || ell < 2 || ell > 64 ||
      f < 0 || f >= ell || (rounds != 8 && rounds != 12 && rounds != 20))
    return BC_EINVAL;
  if (n == 0) return BC_OK;
  if (!x0 || !x1 || !y0 || !y1 || !z0 || !z1 || !seeds) return BC_EINVAL;
  if (!aligned16(x0) || !aligned16(x1) || !aligned16(y0) || !aligned16(y1) || !aligned16(z0) || !aligned16(z1) ||
      (elem_base & 7))
    return BC_EALIGN;
  if (!index_range_ok(elem_base, n)) return BC_ERANGE;  // global indices j < BC_MAX_INDEX
  const size_t nb = n * 8;
  const void* ins[4] = {x0, x1, y0, y1};
  if (overlap(z0, nb, z1, nb)) return BC_EALIAS;
  for (int i = 0; i < 4; ++i)
    if (overlap(z0, nb, ins[i], nb) || overlap(z1, nb, ins[i], nb)) return BC_EALIAS;
  const TP tp{ell == 64 ? ~0ull : ((1ull << ell) - 1ull), (uint32_t)ell};
  const Key k02 = make_key(seeds->s02), k12 = make_key(seeds->s12);
  MulArgs a{x0, x1, y0, y1, z0, z1, (uint64_t)n, elem_base};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return dispatch_rounds(rounds, [&](auto Rc) {
    constexpr int R = decltype(Rc)::value;
    auto fn = k_mul_trc<R>;
    fn<<<grid_for((const void*)fn, (n + 7) / 8, TPB_T), TPB_T, 0, st>>>(a, tp, order, alg, (uint32_t)f, k02, k12);
    return check_launch();
  });
}

int bc_trc_count(int alg, const uint64_t* x, size_t nx, int ell, int k, uint64_t m_base, uint64_t m_count,
                 uint64_t* counts, void* stream) {
  if (!valid_alg(alg, true) || ell < 2 || ell > 64 || k < 1 || k >= ell) return BC_EINVAL;
  if (nx == 0 || m_count == 0) return BC_OK;
  if (!x || !counts) return BC_EINVAL;
  if (!aligned8(x) || !aligned8(counts)) return BC_EALIGN;
  if (overlap(x, nx * 8, counts, nx * 24)) return BC_EALIAS;
  const uint64_t nchunks = (m_count + CNT_CH - 1) / CNT_CH;
  const uint64_t work = (uint64_t)nx * nchunks;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t grid = std::min<uint64_t>(work, (uint64_t)std::max(1, sms) * 8ull);
  k_trc_count<<<(unsigned)grid, CNT_TPB, 0, static_cast<cudaStream_t>(stream)>>>(
      alg, x, (uint64_t)nx, (uint32_t)ell, (uint32_t)k, m_base, m_count, nchunks,
      reinterpret_cast<unsigned long long*>(counts));
  return check_launch();
}

}  // extern "C"
