// intpipe_bench.cu -- measured integer-pipe throughput on this GPU.
//
// Each kernel runs 8 independent dependency chains per thread of one SASS
// instruction class, at full occupancy, and reports thread-ops per second.
// The results set the ALU roofline denominators used in DESIGN.md / bench.py.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o intpipe_bench tools/intpipe_bench.cu
//   ./intpipe_bench            -> one JSON line
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;

#define BODY(OP)                                                      \
  uint32_t v[CH];                                                     \
  _Pragma("unroll") for (int c = 0; c < CH; ++c) v[c] = seed + c * 0x9E3779B9u + threadIdx.x; \
  for (int i = 0; i < ITERS; ++i) {                                   \
    _Pragma("unroll") for (int c = 0; c < CH; ++c) { OP; }            \
  }                                                                   \
  uint32_t acc = 0;                                                   \
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c];         \
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;

__global__ void k_lop3(uint32_t* out, uint32_t seed, uint32_t k) {
  BODY(asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k), "r"(seed)))
}
__global__ void k_shf(uint32_t* out, uint32_t seed, uint32_t k) {
  BODY(asm volatile("shf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(v[c])))
}
__global__ void k_prmt(uint32_t* out, uint32_t seed, uint32_t k) {
  BODY(asm volatile("prmt.b32 %0, %0, %1, 0x2103;" : "+r"(v[c]) : "r"(k)))
}
__global__ void k_iadd3(uint32_t* out, uint32_t seed, uint32_t k) {
  BODY(asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(k)))
}
__global__ void k_imad(uint32_t* out, uint32_t seed, uint32_t k) {
  BODY(asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(k), "r"(seed)))
}
__global__ void k_imadhi(uint32_t* out, uint32_t seed, uint32_t k) {
  BODY(asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(k), "r"(seed)))
}


__global__ void k_mix_lop_imad(uint32_t* out, uint32_t seed, uint32_t k) {
  // one LOP3 and one IMAD per chain per iteration, on separate chains (no dependency between them)
  uint32_t v[CH], w[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c] ^ 0x55u; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k), "r"(seed));
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(w[c]) : "r"(k), "r"(seed));
    }
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c] ^ w[c];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_mix_lop_imadhi(uint32_t* out, uint32_t seed, uint32_t k) {
  uint32_t v[CH], w[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c] ^ 0x55u; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k), "r"(seed));
      asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(w[c]) : "r"(k), "r"(seed));
    }
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c] ^ w[c];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_mix_xsa(uint32_t* out, uint32_t seed, uint32_t k) {
  // ChaCha-like step: x = rotl(x ^ y, 7); y += x  (LOP3, SHF, IMAD.IADD) on 8 chains
  uint32_t v[CH], w[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c] ^ 0x55u; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("xor.b32 %0, %0, %1;" : "+r"(v[c]) : "r"(w[c]));
      asm volatile("shf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(v[c]));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(w[c]) : "r"(v[c]));
    }
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c] ^ w[c];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_viadd(uint32_t* out, uint32_t seed, uint32_t k) {
  BODY(asm volatile("add.u32 %0, %0, 0x3320646e;" : "+r"(v[c])))
}
__global__ void k_mix_lop_viadd(uint32_t* out, uint32_t seed, uint32_t k) {
  uint32_t v[CH], w[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c] ^ 0x55u; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k), "r"(seed));
      asm volatile("add.u32 %0, %0, 0x3320646e;" : "+r"(w[c]));
    }
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c] ^ w[c];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_imadwide(uint32_t* out, uint32_t seed, uint32_t k) {
  uint32_t v[CH];
  uint64_t w[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c]; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c)
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[c]) : "r"(v[c]), "r"(k));
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= (uint32_t)w[c] ^ (uint32_t)(w[c] >> 32);
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_mix_lop_imadwide(uint32_t* out, uint32_t seed, uint32_t k) {
  uint32_t v[CH];
  uint64_t w[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c] ^ 0x55u; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k), "r"(seed));
      asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[c]) : "r"(seed), "r"(k));
    }
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c] ^ (uint32_t)w[c] ^ (uint32_t)(w[c] >> 32);
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_mix_xsa_wide(uint32_t* out, uint32_t seed, uint32_t k) {
  // the ChaCha-like step of k_mix_xsa with the rotate on the FMA pipe:
  // x ^= y; t = x * 2^7 (64-bit); x = lo(t) + hi(t); y += x
  uint32_t v[CH], w[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c] ^ 0x55u; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("xor.b32 %0, %0, %1;" : "+r"(v[c]) : "r"(w[c]));
      asm volatile("{ .reg .b64 t; .reg .b32 lo, hi; mul.wide.u32 t, %0, 128; mov.b64 {lo, hi}, t; add.u32 %0, lo, hi; }"
                   : "+r"(v[c]));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(w[c]) : "r"(v[c]));
    }
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c] ^ w[c];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_mix_xsa_half(uint32_t* out, uint32_t seed, uint32_t k) {
  // half the chains rotate with SHF (ALU), half with the 64-bit multiply (FMA pipe)
  uint32_t v[CH], w[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c] ^ 0x55u; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("xor.b32 %0, %0, %1;" : "+r"(v[c]) : "r"(w[c]));
      if (c & 1)
        asm volatile("{ .reg .b64 t; .reg .b32 lo, hi; mul.wide.u32 t, %0, 128; mov.b64 {lo, hi}, t; add.u32 %0, lo, hi; }"
                     : "+r"(v[c]));
      else
        asm volatile("shf.l.wrap.b32 %0, %0, %0, 7;" : "+r"(v[c]));
      asm volatile("add.u32 %0, %0, %1;" : "+r"(w[c]) : "r"(v[c]));
    }
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c] ^ w[c];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_dp4a(uint32_t* out, uint32_t seed, uint32_t k) {
  BODY(asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(k), "r"(seed)))
}
__global__ void k_mix_lop_dp4a(uint32_t* out, uint32_t seed, uint32_t k) {
  uint32_t v[CH], w[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c] ^ 0x55u; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k), "r"(seed));
      asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(w[c]) : "r"(k), "r"(seed));
    }
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c] ^ w[c];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_mix_lop_imad_dp4a(uint32_t* out, uint32_t seed, uint32_t k) {
  // 2 LOP3 : 1 IMAD : 1 DP4A -- does DP4A share the FMA pipe with IMAD?
  uint32_t v[CH], w[CH], x[CH];
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { v[c] = seed + c * 0x9E3779B9u + threadIdx.x; w[c] = v[c] ^ 0x55u; x[c] = w[c] + 7u; }
  for (int i = 0; i < ITERS; ++i) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(k), "r"(seed));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x69;" : "+r"(v[c]) : "r"(k), "r"(seed));
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(w[c]) : "r"(k), "r"(seed));
      asm volatile("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(k), "r"(seed));
    }
  }
  uint32_t acc = 0;
  _Pragma("unroll") for (int c = 0; c < CH; ++c) acc ^= v[c] ^ w[c] ^ x[c];
  if (acc == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_lds(uint32_t* out, uint32_t seed, uint32_t k) {
  // random 4-B shared loads (the table kernels' access pattern): 32 lanes, random words
  __shared__ uint32_t tab[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) tab[i] = i * 0x9E3779B9u;
  __syncthreads();
  BODY(v[c] = tab[(v[c] ^ k) & 8191u])
}

template <typename K>
double rate(K kern, int ops_per_iter, int blocks, int threads) {
  uint32_t* out;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  kern<<<blocks, threads>>>(out, 1u, 3u);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) kern<<<blocks, threads>>>(out, 1u + r, 3u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  const double ops = (double)reps * blocks * threads * ITERS * CH * ops_per_iter;
  return ops / (ms * 1e-3) / 1e12;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int threads = 256, blocks = sms * 8;
  printf("{\"sms\": %d, \"clock_khz_attr\": %d", sms, clk);
  printf(", \"lop3_tops\": %.3f", rate(k_lop3, 1, blocks, threads));
  printf(", \"shf_tops\": %.3f", rate(k_shf, 1, blocks, threads));
  printf(", \"prmt_tops\": %.3f", rate(k_prmt, 1, blocks, threads));
  printf(", \"imad_tops\": %.3f", rate(k_imad, 1, blocks, threads));
  printf(", \"imad_hi_tops\": %.3f", rate(k_imadhi, 1, blocks, threads));
  printf(", \"viadd_tops\": %.3f", rate(k_viadd, 1, blocks, threads));
  printf(", \"lop3+viadd_tops\": %.3f", rate(k_mix_lop_viadd, 2, blocks, threads));
  printf(", \"lop3+imad_tops\": %.3f", rate(k_mix_lop_imad, 2, blocks, threads));
  printf(", \"lop3+imadhi_tops\": %.3f", rate(k_mix_lop_imadhi, 2, blocks, threads));
  printf(", \"xor_rot_add_tops\": %.3f", rate(k_mix_xsa, 3, blocks, threads));
  printf(", \"imad_wide_tops\": %.3f", rate(k_imadwide, 1, blocks, threads));
  printf(", \"lop3+imadwide_tops\": %.3f", rate(k_mix_lop_imadwide, 2, blocks, threads));
  // the two ChaCha-like variants in the same unit as xor_rot_add: 3 algorithmic ops per step
  printf(", \"xor_rotwide_add_tops\": %.3f", rate(k_mix_xsa_wide, 3, blocks, threads));
  printf(", \"xor_rot_add_half_wide_tops\": %.3f", rate(k_mix_xsa_half, 3, blocks, threads));
  printf(", \"dp4a_tops\": %.3f", rate(k_dp4a, 1, blocks, threads));
  printf(", \"lop3+dp4a_tops\": %.3f", rate(k_mix_lop_dp4a, 2, blocks, threads));
  printf(", \"2lop3+imad+dp4a_tops\": %.3f", rate(k_mix_lop_imad_dp4a, 4, blocks, threads));
  printf(", \"lds_random_tops\": %.3f", rate(k_lds, 1, blocks, threads));
  printf("}\n");
  return 0;
}
