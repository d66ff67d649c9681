// bc_host.cu -- host-side utilities and the parameter / error entry points of the C ABI.
#include <cstring>
#include <mutex>

#include "bc_common.cuh"

namespace {
thread_local int g_last_cuda = 0;

bool is_prime(uint64_t v) {
  if (v < 2) return false;
  for (uint64_t d = 2; d * d <= v; ++d)
    if (v % d == 0) return false;
  return true;
}

uint32_t factorial(uint32_t s) {
  uint32_t f = 1;
  for (uint32_t i = 2; i <= s; ++i) f *= i;
  return f;
}
}  // namespace

namespace bc {
namespace host {

int cuda_rc(cudaError_t e) {
  if (e != cudaSuccess) {
    g_last_cuda = (int)e;
    return BC_ECUDA;
  }
  return BC_OK;
}

int check_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_last_cuda = (int)e;
    return BC_ECUDA;
  }
  return BC_OK;
}

// Persistent grid: min(#work blocks, #SM x resident blocks per SM), cached per (kernel, device).
int grid_for(const void* fn, uint64_t nthreads_work, int tpb, size_t smem) {
  struct Entry {
    const void* fn;
    int dev;
    int cap;
  };
  static std::mutex mu;
  static Entry cache[512];
  static int ncache = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int cap = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < ncache; ++i)
      if (cache[i].fn == fn && cache[i].dev == dev) {
        cap = cache[i].cap;
        break;
      }
    if (!cap) {
      int sms = 0, occ = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, tpb, smem);
      cap = std::max(1, sms) * std::max(1, occ);
      if (ncache < 512) cache[ncache++] = Entry{fn, dev, cap};
    }
  }
  const uint64_t want = (nthreads_work + (uint64_t)tpb - 1) / (uint64_t)tpb;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)cap));
}

// Opt-in to more than 48 KB of dynamic shared memory, once per (kernel, device).
int allow_smem(const void* fn, size_t bytes) {
  struct Entry {
    const void* fn;
    int dev;
  };
  static std::mutex mu;
  static Entry done[256];
  static int ndone = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < ndone; ++i)
    if (done[i].fn == fn && done[i].dev == dev) return BC_OK;
  const int rc = cuda_rc(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  if (rc) return rc;
  if (ndone < 256) done[ndone++] = Entry{fn, dev};
  return BC_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool aligned8(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7u) == 0; }

bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  if (!a || !b || !na || !nb) return false;
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}

bool index_range_ok(uint64_t base, size_t n) { return base <= BC_MAX_INDEX && (uint64_t)n <= BC_MAX_INDEX - base; }

int check_params(const bc_params* prm) {
  if (!prm) return BC_EINVAL;
  bc_params ref;
  const int rc = bc_params_init(&ref, prm->ell, prm->lx, prm->f, prm->mode, prm->rounds);
  if (rc) return rc;
  if (ref.w != prm->w || ref.p != prm->p || ref.slots != prm->slots || ref.tape != prm->tape) return BC_EINVAL;
  return BC_OK;
}

KP make_kp(const bc_params* prm) {
  KP kp;
  kp.ymask = prm->ell == 64 ? ~0ull : ((1ull << prm->ell) - 1ull);
  kp.f = (uint32_t)prm->f;
  kp.fsh = (uint32_t)prm->f & 31u;
  kp.fhi = prm->f >= 32 ? 1u : 0u;
  kp.w = prm->w;
  kp.p = (uint32_t)prm->p;  // only used by the p <= 257 tapes
  kp.S = prm->slots;
  kp.lx = (uint32_t)prm->lx;
  kp.wmask = (uint32_t)((1ull << prm->w) - 1ull);
  kp.one = 1u;
  if (prm->tape != BC_TAPE_LARGE) {
    kp.fact = factorial(prm->slots);
    kp.perm_lim = (uint32_t)((0x80000000ull / kp.fact) * kp.fact);
    // pair tape (p <= 131): d = (p-1) p < 2^15; with k = floor(log2 d), M = ceil(2^(32+k) / d) < 2^32
    // (d is never a power of two) overshoots by e < d, and u e < 2^28 2^(k+1) < 2^(32+k): exact for u < 2^28
    kp.pair_d = (kp.p - 1u) * kp.p;
    kp.pair_lim = ((1u << 28) / kp.pair_d) * kp.pair_d;
    kp.pair_sh = 31u - (uint32_t)__builtin_clz(kp.pair_d);
    kp.pair_mag = (uint32_t)(((1ull << (32 + kp.pair_sh)) + kp.pair_d - 1) / kp.pair_d);
    // x / d for x < 2^16, d <= 257: ceil(2^32 / d) overshoots 2^32/d by e < 1, and x e / 2^32 < 1/d
    kp.mag_p = (uint32_t)(((1ull << 32) + kp.p - 1) / kp.p);
    kp.mag_q = (uint32_t)(((1ull << 32) + kp.p - 2) / (kp.p - 1u));
    // x / S! for x < 2^31 (round-up method, l = ceil(log2 S!)): m = ceil(2^(31+l) / S!) < 2^32
    uint32_t l = 0;
    while ((1ull << l) < kp.fact) ++l;
    kp.mag_f = (uint32_t)(((1ull << (31 + l)) + kp.fact - 1) / kp.fact);
    kp.sh_f = l - 1;
  }
  return kp;
}

KPL make_kpl(const bc_params* prm) {
  using u128 = unsigned __int128;
  KPL k{};
  const uint64_t p = prm->p, q = p - 1;
  k.ymask = prm->ell == 64 ? ~0ull : ((1ull << prm->ell) - 1ull);
  k.wmask = (1ull << prm->w) - 1ull;
  k.p = p;
  uint64_t inv = p;  // p^-1 mod 2^64 by Newton (p odd: correct to 3 bits, doubling per step)
  for (int i = 0; i < 5; ++i) inv *= 2ull - p * inv;
  k.pinv = inv;
  k.mu_p = ~0ull / p;
  k.mu_q = ~0ull / q;
  k.qinv_p = 1.0 / (double)p;
  k.qoff_p = -(4503599627370496.0 + (double)((p - 1) / 2));
  k.s_q = 0;
  while (((q >> k.s_q) & 1ull) == 0) ++k.s_q;
  const uint64_t qo = q >> k.s_q;  // odd part of p - 1
  k.qinv_q = 1.0 / (double)qo;
  k.qoff_q = -(4503599627370496.0 + (double)((qo - 1) / 2));
  const u128 two48 = (u128)1 << 48;  // the large tape's draws are 48-bit
  const u128 pl = two48 / p * p, ql = two48 / q * q;
  k.plim = (uint64_t)(pl - 1);  // accept u <= lim - 1; 2^48 - 1 when q | 2^48 (nothing rejects)
  k.qlim = (uint64_t)(ql - 1);
  k.wm32 = (uint32_t)((1ull << prm->w) - 1ull);
  k.two_w = (1ull << prm->w) % p;
  k.off1 = p - (1ull << prm->w);
  k.f = (uint32_t)prm->f;
  k.w = prm->w;
  k.S = prm->slots;
  return k;
}

KeyPre make_keypre(const uint8_t* s, uint64_t label) {
  KeyPre p;
  std::memcpy(p.k, s, 32);
  p.l0 = (uint32_t)label;
  p.l1 = (uint32_t)(label >> 32);
  auto rotl = [](uint32_t v, int n) { return (v << n) | (v >> (32 - n)); };
  auto qr = [&](uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {  // RFC 8439 sec. 2.1
    a += b; d ^= a; d = rotl(d, 16);
    c += d; b ^= c; b = rotl(b, 12);
    a += b; d ^= a; d = rotl(d, 8);
    c += d; b ^= c; b = rotl(b, 7);
  };
  uint32_t x2 = 0x79622d32u, x6 = p.k[2], x10 = p.k[6], x14 = p.l0;
  uint32_t x3 = 0x6b206574u, x7 = p.k[3], x11 = p.k[7], x15 = p.l1;
  qr(x2, x6, x10, x14);
  qr(x3, x7, x11, x15);
  const uint32_t c[8] = {x2, x6, x10, x14, x3, x7, x11, x15};
  std::memcpy(p.c, c, sizeof c);
  uint32_t x1 = 0x3320646eu, x5 = p.k[1], x9 = p.k[5], x13 = 0u;  // column 1 with a zero counter high word
  qr(x1, x5, x9, x13);
  const uint32_t c1[4] = {x1, x5, x9, x13};
  std::memcpy(p.c1, c1, sizeof c1);
  return p;
}

Key make_key(const uint8_t* s) {
  Key k;
  std::memcpy(k.k, s, 32);  // little-endian host: words are the LE u32 of the seed
  k.m7 = 1u << 7;
  return k;
}

}  // namespace host
}  // namespace bc

extern "C" {

int bc_version(void) { return 301; }

int bc_last_cuda_error(void) { return g_last_cuda; }

const char* bc_strerror(int code) {
  switch (code) {
    case BC_OK: return "ok";
    case BC_EINVAL: return "invalid parameter";
    case BC_ERANGE: return "key-bit window does not fit (need f + lx + w <= ell), or elem_base + n > BC_MAX_INDEX";
    case BC_EALIGN: return "pointer misaligned (16 B for u64 arrays) or elem_base not a multiple of 8";
    case BC_ECUDA: return "CUDA launch error (see bc_last_cuda_error)";
    case BC_EALIAS: return "output overlaps an input";
    default: return "unknown error";
  }
}

int bc_params_init(bc_params* out, int ell, int lx, int f, int mode, int rounds) {
  if (!out) return BC_EINVAL;
  if (ell < 2 || ell > 64 || lx < 2 || lx > 31 || f < 0 || (mode != BC_MODE_GUARD && mode != BC_MODE_LITERAL) ||
      (rounds != 8 && rounds != 12 && rounds != 20))
    return BC_EINVAL;
  const uint32_t w = (uint32_t)(mode == BC_MODE_GUARD ? lx + 1 : lx);
  if ((uint64_t)f + (uint64_t)lx + w > (uint64_t)ell) return BC_ERANGE;
  uint64_t p = (1ull << w) + 1ull;  // smallest prime > 2^w (reading C7)
  while (!is_prime(p)) ++p;
  bc_params r;
  r.ell = ell;
  r.lx = lx;
  r.f = f;
  r.mode = mode;
  r.rounds = rounds;
  r.w = w;
  r.p = p;
  r.slots = (uint32_t)lx + 1u;
  r.tape = (p == 257u && r.slots == 8u)   ? BC_TAPE_COMPACT
           : (p == 131u && r.slots == 8u) ? BC_TAPE_COMPACT_LIT
           : (lx <= 7 ? BC_TAPE_PAIR : BC_TAPE_LARGE);
  *out = r;
  return BC_OK;
}

}  // extern "C"
