// bc_common.cuh -- shared device templates and host utilities of libbicoptor.
//
// Thread <-> data mapping: one thread owns a group of 8
// consecutive elements.  That is the natural unit of the PRG: the compact
// seed01 tape is 24 B per element (3 ChaCha blocks per group: two of part A,
// one of part B), the pair tape 32 B (4 blocks per group), and every 8-B
// per-element stream of seed02 / seed12 is exactly one block per group, so no
// keystream byte is generated twice and no keystream is exchanged between
// threads.  Share vectors move as 4 x 16-B vector accesses per party per group.
// Grids are persistent: (#SM x resident blocks) CTAs in a grid-stride loop.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "bc_compact.cuh"
#include "bc_device.cuh"
#include "bc_large.cuh"
#include "bicoptor.h"

namespace bc {

constexpr int TPB = 256;
#ifndef BC_FUSED_MINB
#define BC_FUSED_MINB 2
#endif
constexpr int FUSED_MINB = BC_FUSED_MINB;  // resident CTAs per SM the fused kernels are compiled for

__device__ __forceinline__ uint64_t u64_of(const uint32_t (&B)[16], int e) {
  return (uint64_t)B[2 * e] | ((uint64_t)B[2 * e + 1] << 32);
}

// Two consecutive elements (one 16-B vector per party); zero past n.
__device__ __forceinline__ ulonglong2 load2(const uint64_t* __restrict__ p, uint64_t i, uint64_t n) {
  if (i + 1 < n) return __ldg(reinterpret_cast<const ulonglong2*>(p + i));
  return make_ulonglong2(i < n ? __ldg(p + i) : 0ull, 0ull);
}

__device__ __forceinline__ uint64_t load_hi8(const uint8_t* hi, uint64_t i0, uint32_t cnt) {
  if (!hi) return 0;
  if (cnt == 8) return __ldg(reinterpret_cast<const unsigned long long*>(hi + i0));
  uint64_t v = 0;
  for (uint32_t e = 0; e < cnt; ++e) v |= (uint64_t)hi[i0 + e] << (8 * e);
  return v;
}

// ---- host utilities (bc_host.cu) ------------------------------------------
namespace host {
int check_launch();                                  // cudaGetLastError -> BC_OK / BC_ECUDA
int cuda_rc(cudaError_t e);                          // records e for bc_last_cuda_error
int grid_for(const void* fn, uint64_t nthreads_work, int tpb = TPB, size_t smem = 0);  // persistent grid size
KPL make_kpl(const bc_params* prm);                  // large-tape constants (p < 2^33)
int allow_smem(const void* fn, size_t bytes);       // dynamic shared memory above 48 KB (cached)
bool aligned16(const void* p);
bool aligned8(const void* p);
bool overlap(const void* a, size_t na, const void* b, size_t nb);
bool index_range_ok(uint64_t base, size_t n);       // [base, base + n) within [0, BC_MAX_INDEX]
int check_params(const bc_params* prm);              // re-derives and compares
KP make_kp(const bc_params* prm);
Key make_key(const uint8_t* s);
KeyPre make_keypre(const uint8_t* s, uint64_t label);  // chacha_pre's first-round precomputation

template <typename F>
int dispatch_rounds(int rounds, F&& f) {
  switch (rounds) {
    case 8: return f(std::integral_constant<int, 8>{});
    case 12: return f(std::integral_constant<int, 12>{});
    case 20: return f(std::integral_constant<int, 20>{});
    default: return BC_EINVAL;
  }
}
}  // namespace host
}  // namespace bc
