/* bicoptor_ref.c -- scalar C reference of Bicoptor 2.0 DReLU (Alg 7) and ReLU (Alg 8).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load it (through oracle/cref.py).  It shares
 * no code, header, table or constant generator with the CUDA path
 * (paper_2309_04909_b200/csrc); it is a second, plain transcription of the same
 * algorithms as oracle/bicoptor.py, one element at a time, in the paper's order.
 * Its own pins: the RFC 8439 block (tests/test_oracle_cref.py) and bit-exact
 * agreement with the numpy oracle, which is pinned against the paper
 * (tests/test_oracle_*.py).
 *
 * Citations: P:n = line n of the paper's LaTeX source; Cn = the
 * readings listed in DESIGN.md sec. 3; the PRG tape layout is DESIGN.md sec. 4.
 *
 * Per element j (a global index) and party b in {0, 1}:
 *   Alg 7
 *     1  t from seed01's tape                        2  s_b = (-1)^t [x]_b mod 2^ell
 *     3  u_i = trc(s_b, f+i, ell-w-f-i), i = 0..lx   (Alg 5; C1-C5)
 *     4  v_i = u_i + u_{i+1} - 1, v_lx = u_lx - 1    (mod 2^w; P0 adds the -1, C8)
 *     5  v'_i = modswitch(v_i)                        (Alg 6)
 *     6  shuffle with Pi                              (Fisher-Yates, C9)
 *     7  w_m = v'_m r_m mod p                         8  W_m = w_m +- rho_m mod p (C11)
 *     9  P2: z = [exists m: W0_m + W1_m = 0 mod p]    10 [D']_0 = seed02 stream, [D']_1 = z - [D']_0
 *    11  y_b = t + (1-2t)[D']_b (P0 adds t), mod 2^ell
 *   Alg 8: triple (a, b, c) from seed02 / seed12 (C24), d = x - a opened,
 *     e = z - b from P2, y_b = t [x]_b + (1-2t)(de + d[b]_b + e[a]_b + [c]_b) (P0 adds de).
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC -o libbcref.so bicoptor_ref.c   (oracle/cref.py)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------------------
 * ChaCha_R block, RFC 8439 sec. 2.3 (reading C19), state words 12-13 = 64-bit block
 * counter, 14-15 = 64-bit stream label.
 * ---------------------------------------------------------------------------------- */
static uint32_t rotl32(uint32_t v, int n) { return (v << n) | (v >> (32 - n)); }

static void quarter(uint32_t *x, int a, int b, int c, int d) {
  x[a] += x[b]; x[d] ^= x[a]; x[d] = rotl32(x[d], 16);
  x[c] += x[d]; x[b] ^= x[c]; x[b] = rotl32(x[b], 12);
  x[a] += x[b]; x[d] ^= x[a]; x[d] = rotl32(x[d], 8);
  x[c] += x[d]; x[b] ^= x[c]; x[b] = rotl32(x[b], 7);
}

static uint32_t le32(const uint8_t *p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

void bcref_chacha_block(const uint8_t key[32], uint64_t label, uint64_t counter, int rounds, uint8_t out[64]) {
  uint32_t st[16], x[16];
  st[0] = 0x61707865u; st[1] = 0x3320646eu; st[2] = 0x79622d32u; st[3] = 0x6b206574u;
  for (int i = 0; i < 8; ++i) st[4 + i] = le32(key + 4 * i);
  st[12] = (uint32_t)counter; st[13] = (uint32_t)(counter >> 32);
  st[14] = (uint32_t)label; st[15] = (uint32_t)(label >> 32);
  memcpy(x, st, sizeof x);
  for (int r = 0; r < rounds; r += 2) {
    quarter(x, 0, 4, 8, 12); quarter(x, 1, 5, 9, 13); quarter(x, 2, 6, 10, 14); quarter(x, 3, 7, 11, 15);
    quarter(x, 0, 5, 10, 15); quarter(x, 1, 6, 11, 12); quarter(x, 2, 7, 8, 13); quarter(x, 3, 4, 9, 14);
  }
  for (int i = 0; i < 16; ++i) {
    const uint32_t v = x[i] + st[i];
    out[4 * i] = (uint8_t)v; out[4 * i + 1] = (uint8_t)(v >> 8);
    out[4 * i + 2] = (uint8_t)(v >> 16); out[4 * i + 3] = (uint8_t)(v >> 24);
  }
}

/* Bytes [off, off + len) of the keystream (key, label): the concatenation of the blocks
 * with counters 0, 1, 2, ...  Element j of a stride-s stream owns [s j, s j + s). */
static void ks_bytes(const uint8_t key[32], uint64_t label, int rounds, uint64_t off, unsigned len, uint8_t *dst) {
  uint8_t blk[64];
  uint64_t cur = ~0ull;
  for (unsigned i = 0; i < len; ++i) {
    const uint64_t pos = off + i;
    if (pos / 64 != cur) {
      cur = pos / 64;
      bcref_chacha_block(key, label, cur, rounds, blk);
    }
    dst[i] = blk[pos % 64];
  }
}

static uint64_t label_of(const char *s) { /* 8 ASCII bytes, little endian */
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | (uint8_t)s[i];
  return v;
}

/* Sequential words of a fallback stream (reading C10). */
typedef struct {
  const uint8_t *key;
  uint64_t label, ctr;
  int rounds, pos;
  uint8_t blk[64];
} fbstream;

static void fb_init(fbstream *fb, const uint8_t *key, const char *lab, uint64_t ctr0, int rounds) {
  fb->key = key; fb->label = label_of(lab); fb->ctr = ctr0; fb->rounds = rounds; fb->pos = 64;
}
static uint32_t fb_u32(fbstream *fb) {
  if (fb->pos == 64) { bcref_chacha_block(fb->key, fb->label, fb->ctr++, fb->rounds, fb->blk); fb->pos = 0; }
  const uint32_t v = le32(fb->blk + fb->pos);
  fb->pos += 4;
  return v;
}
static uint64_t fb_u64(fbstream *fb) {
  if (fb->pos == 64) { bcref_chacha_block(fb->key, fb->label, fb->ctr++, fb->rounds, fb->blk); fb->pos = 0; }
  const uint64_t v = (uint64_t)le32(fb->blk + fb->pos) | ((uint64_t)le32(fb->blk + fb->pos + 4) << 32);
  fb->pos += 8;
  return v;
}

/* ------------------------------------------------------------------------------------
 * Parameters (reading C5-C7): w = lx + 1 (guard) or lx (literal); p = smallest prime
 * > 2^w; S = lx + 1 ladder slots.  Tape layout: compact (p = 257,
 * S = 8), pair (other lx <= 7), large (lx >= 8).
 * ---------------------------------------------------------------------------------- */
enum { COMPACT = 0, PAIR = 1, LARGE = 2 };
typedef struct {
  int ell, lx, f, w, S, rounds, layout;
  uint64_t p, ymask, rinv; /* rinv = 2^-64 mod p (large tape) */
} prm_t;

static int is_prime(uint64_t n) {
  if (n < 2) return 0;
  for (uint64_t d = 2; d * d <= n; ++d)
    if (n % d == 0) return 0;
  return 1;
}

static uint64_t mask_bits(int bits) { return bits >= 64 ? ~0ull : ((1ull << bits) - 1ull); }

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)(((u128)a * b) % p); }

static int prm_make(prm_t *P, int ell, int lx, int f, int literal, int rounds) {
  if (ell < 2 || ell > 64 || lx < 2 || lx > 31 || f < 0) return -1;
  if (rounds != 8 && rounds != 12 && rounds != 20) return -1;
  P->ell = ell; P->lx = lx; P->f = f; P->rounds = rounds;
  P->w = literal ? lx : lx + 1;
  if (f + lx + P->w > ell) return -1;
  P->S = lx + 1;
  uint64_t p = (1ull << P->w) + 1;
  while (!is_prime(p)) ++p;
  P->p = p;
  P->ymask = mask_bits(ell);
  P->layout = (p == 257 && P->S == 8) ? COMPACT : (lx <= 7 ? PAIR : LARGE);
  uint64_t inv2 = (p + 1) / 2, r = 1; /* (2^-1)^64 mod p */
  for (int i = 0; i < 64; ++i) r = mulmod(r, inv2, p);
  P->rinv = r;
  return 0;
}

/* ------------------------------------------------------------------------------------
 * The seed01 tape of one element: t (step 1), Fisher-Yates partners k_m (step 6),
 * masks r_m in Z_p^* (step 7), reshares rho_m in Z_p (step 8).  DESIGN.md sec. 4.
 * ---------------------------------------------------------------------------------- */
typedef struct {
  uint32_t t;
  uint32_t k[32];
  uint64_t r[32], rho[32];
} tape_t;

static uint64_t factorial(int S) {
  uint64_t f = 1;
  for (int i = 2; i <= S; ++i) f *= (uint64_t)i;
  return f;
}

/* k_m = q mod (m+1), q /= (m+1), for m = S-1 .. 1 (reading C9). */
static void perm_digits(uint64_t q, int S, uint32_t *k) {
  q %= factorial(S);
  k[0] = 0;
  for (int m = S - 1; m >= 1; --m) {
    k[m] = (uint32_t)(q % (uint64_t)(m + 1));
    q /= (uint64_t)(m + 1);
  }
}

static void tape_compact(const prm_t *P, const uint8_t *s01, uint64_t j, tape_t *tp) {
  uint8_t a[16], b[8];
  ks_bytes(s01, label_of("bc2.tpa1"), P->rounds, 16 * j, 16, a);  /* part A: 16 B at 16 j */
  ks_bytes(s01, label_of("bc2.tpb1"), P->rounds, 8 * j, 8, b);    /* part B:  8 B at  8 j */
  const uint32_t T0 = le32(a);
  uint32_t idx = T0 & 0x7FFFFFFFu;
  uint32_t words[3] = {le32(a + 12), le32(b), le32(b + 4)};
  const uint32_t perm_lim = 53261u * 40320u, rho_lim = 253u * 257u * 257u * 257u;
  fbstream fb;
  fb_init(&fb, s01, "bc2.fb01", j * 256, P->rounds);
  if (idx >= perm_lim) {            /* fallback order: the index, then the reshare words */
    do idx = fb_u32(&fb) & 0x7FFFFFFFu; while (idx >= perm_lim);
  }
  for (int k = 0; k < 3; ++k)
    while (words[k] >= rho_lim) words[k] = fb_u32(&fb);
  tp->t = T0 >> 31;
  perm_digits(idx, 8, tp->k);
  for (int m = 0; m < 8; ++m) tp->r[m] = 1 + (uint64_t)a[4 + m];   /* exactly uniform on Z_257^* */
  for (int m = 0; m < 8; ++m) {                                     /* base-257 digits, LSB first */
    uint32_t w = words[m / 3];
    for (int i = 0; i < m % 3; ++i) w /= 257u;
    tp->rho[m] = w % 257u;
  }
}

static void tape_pair(const prm_t *P, const uint8_t *s01, uint64_t j, tape_t *tp) {
  uint8_t e[32];
  ks_bytes(s01, label_of("bc2.tpp1"), P->rounds, 32 * j, 32, e);   /* 32 B at 32 j */
  const int S = P->S;
  const uint64_t p = P->p, d = (p - 1) * p, lim = ((1ull << 28) / d) * d;
  const uint64_t fact = factorial(S), plim = ((1ull << 31) / fact) * fact;
  const uint32_t T0 = le32(e);
  uint64_t idx = T0 & 0x7FFFFFFFu;
  uint64_t u[8];
  for (int m = 0; m < S; ++m) {     /* bits [32 + 28 m, 32 + 28 m + 28) of the 32 bytes, LSB first */
    uint64_t v = 0;
    for (int bit = 0; bit < 28; ++bit) {
      const int pos = 32 + 28 * m + bit;
      v |= (uint64_t)((e[pos / 8] >> (pos % 8)) & 1u) << bit;
    }
    u[m] = v;
  }
  fbstream fb;
  fb_init(&fb, s01, "bc2.fb01", j * 256, P->rounds);
  if (idx >= plim) {
    do idx = fb_u32(&fb) & 0x7FFFFFFFu; while (idx >= plim);
  }
  for (int m = 0; m < S; ++m)
    while (u[m] >= lim) u[m] = fb_u32(&fb) & 0x0FFFFFFFu;
  tp->t = T0 >> 31;
  perm_digits(idx, S, tp->k);
  for (int m = 0; m < S; ++m) {
    const uint64_t x = u[m] % d;    /* a uniform pair (x mod (p-1), x div (p-1)) */
    tp->r[m] = 1 + x % (p - 1);
    tp->rho[m] = x / (p - 1);
  }
}

static void tape_large(const prm_t *P, const uint8_t *s01, uint64_t j, tape_t *tp) {
  uint8_t e[448];
  ks_bytes(s01, label_of("bc2.tpL2"), P->rounds, 448 * j, 448, e);  /* 7 blocks at 448 j */
  const int S = P->S;
  const uint64_t p = P->p, m48 = (1ull << 48) - 1;
  const uint64_t rlim = ((1ull << 48) / (p - 1)) * (p - 1), plim = ((1ull << 48) / p) * p;
  fbstream fb;
  fb_init(&fb, s01, "bc2.fbL2", j << 20, P->rounds);
  tp->t = e[0] & 1u;                                   /* h[0] & 1 */
  tp->k[0] = 0;
  for (int m = S - 1; m >= 1; --m) {                   /* draw of slot m: h[S - m] */
    uint64_t h = (uint64_t)e[2 * (S - m)] | ((uint64_t)e[2 * (S - m) + 1] << 8);
    const uint64_t hl = (65536 / (uint64_t)(m + 1)) * (uint64_t)(m + 1);
    while (h >= hl) h = fb_u64(&fb) & 0xFFFFu;
    tp->k[m] = (uint32_t)(h % (uint64_t)(m + 1));
  }
  for (int m = 0; m < S; ++m) {
    const int om = 64 + 96 * (m / 8) + 6 * (m % 8);   /* from the start of block 1 */
    uint64_t ur = 0, uh = 0;
    for (int i = 0; i < 6; ++i) {
      ur |= (uint64_t)e[om + i] << (8 * i);
      uh |= (uint64_t)e[om + 48 + i] << (8 * i);
    }
    while (ur >= rlim) ur = fb_u64(&fb) & m48;
    tp->r[m] = mulmod(1 + ur % (p - 1), P->rinv, p);  /* (1 + u mod (p-1)) 2^-64 mod p (C28) */
    while (uh >= plim) uh = fb_u64(&fb) & m48;
    tp->rho[m] = uh % p;
  }
}

static void tape(const prm_t *P, const uint8_t *s01, uint64_t j, tape_t *tp) {
  if (P->layout == COMPACT) tape_compact(P, s01, j, tp);
  else if (P->layout == PAIR) tape_pair(P, s01, j, tp);
  else tape_large(P, s01, j, tp);
}

/* ------------------------------------------------------------------------------------
 * Alg 5 / Alg 6 for one party.
 * ---------------------------------------------------------------------------------- */
/* Alg 5 (C1-C4): P0 cut(s, k1, k2) = bits [k1, ell-k2) of s; P1 -cut(-s, k1, k2),
 * both mod 2^(ell-k1-k2). */
static uint64_t trc_mid(const prm_t *P, int party, uint64_t s, int k1, int k2) {
  const int lp = P->ell - k1 - k2;
  const uint64_t lm = mask_bits(lp);
  if (party == 0) return (s >> k1) & lm;
  const uint64_t ns = (0ull - s) & P->ymask;
  return (0ull - ((ns >> k1) & lm)) & lm;
}

/* Alg 6: P0: 2^w mod p if v = 0 else v mod p; P1: p + v - 2^w mod p. */
static uint64_t modswitch(const prm_t *P, int party, uint64_t v) {
  const uint64_t two_w = 1ull << P->w;
  if (party == 0) return v == 0 ? two_w % P->p : v % P->p;
  return (P->p + v - two_w) % P->p;
}

/* Alg 7 steps 3-5 on s (no blinding): v'_0 .. v'_lx. */
static void ladder_modswitch(const prm_t *P, int party, uint64_t s, uint64_t *vp) {
  uint64_t u[33];
  const uint64_t wm = mask_bits(P->w), one = party == 0 ? 1 : 0;
  for (int i = 0; i <= P->lx; ++i) u[i] = trc_mid(P, party, s, P->f + i, P->ell - P->w - P->f - i);  /* step 3 */
  for (int i = 0; i <= P->lx; ++i) {                                                                 /* step 4 */
    const uint64_t nxt = i < P->lx ? u[i + 1] : 0;
    vp[i] = modswitch(P, party, (u[i] + nxt - one) & wm);                                          /* step 5 */
  }
}

/* Alg 7 steps 1-8 for P0 / P1: the message W (S slots in Z_p). */
static void drelu_send(const prm_t *P, int party, uint64_t xb, const tape_t *tp, uint64_t *W) {
  const uint64_t s = tp->t ? (0ull - xb) & P->ymask : xb;          /* steps 1-2 */
  uint64_t v[32];
  ladder_modswitch(P, party, s, v);                                  /* steps 3-5 */
  for (int m = P->S - 1; m >= 1; --m) {                              /* step 6 */
    const uint64_t a = v[m];
    v[m] = v[tp->k[m]];
    v[tp->k[m]] = a;
  }
  for (int m = 0; m < P->S; ++m) {
    const uint64_t wv = mulmod(v[m], tp->r[m], P->p);                /* step 7 */
    W[m] = party == 0 ? (wv + tp->rho[m]) % P->p                    /* step 8 */
                      : (wv + P->p - tp->rho[m]) % P->p;
  }
}

/* Alg 7 step 9. */
static uint64_t zero_test(const prm_t *P, const uint64_t *W0, const uint64_t *W1) {
  uint64_t z = 0;
  for (int m = 0; m < P->S; ++m)
    if ((W0[m] + W1[m]) % P->p == 0) z = 1;
  return z;
}

static uint64_t stream_u64(const uint8_t *key, const char *lab, int rounds, uint64_t j) {
  uint8_t b[8];
  ks_bytes(key, label_of(lab), rounds, 8 * j, 8, b);
  return (uint64_t)le32(b) | ((uint64_t)le32(b + 4) << 32);
}

/* Alg 7 step 11: t + (1-2t) [D']_b, P0 adds t (C8). */
static uint64_t drelu_finish(const prm_t *P, int party, uint32_t t, uint64_t Db) {
  const uint64_t sg = t ? (0ull - Db) & P->ymask : Db;
  return party == 0 ? (sg + t) & P->ymask : sg;
}

static void one_element(const prm_t *P, const uint8_t *s01, const uint8_t *s02, const uint8_t *s12, uint64_t x0,
                        uint64_t x1, uint64_t j, int relu, uint64_t *y0, uint64_t *y1, uint64_t *W0, uint64_t *W1) {
  const uint64_t M = P->ymask;
  const int R = P->rounds;
  tape_t tp;
  tape(P, s01, j, &tp);
  drelu_send(P, 0, x0, &tp, W0);                                   /* P0 -> P2 */
  drelu_send(P, 1, x1, &tp, W1);                                   /* P1 -> P2 */
  const uint64_t z = zero_test(P, W0, W1);                         /* P2, step 9 */
  if (!relu) {
    const uint64_t D0 = stream_u64(s02, "bc2.resp", R, j) & M;   /* step 10 (C12) */
    const uint64_t D1 = (z - D0) & M;
    *y0 = drelu_finish(P, 0, tp.t, D0);
    *y1 = drelu_finish(P, 1, tp.t, D1);
    return;
  }
  /* Alg 8 */
  const uint64_t a0 = stream_u64(s02, "bc2.ta02", R, j) & M, b0 = stream_u64(s02, "bc2.tb02", R, j) & M;
  const uint64_t c0 = stream_u64(s02, "bc2.tc02", R, j) & M;
  const uint64_t a1 = stream_u64(s12, "bc2.ta12", R, j) & M, b1 = stream_u64(s12, "bc2.tb12", R, j) & M;
  const uint64_t c1 = ((a0 + a1) * (b0 + b1) - c0) & M;            /* P2's [c]_1 (C20, C24) */
  const uint64_t d0 = (x0 - a0) & M, d1 = (x1 - a1) & M;            /* step 4: [d]_b = [x]_b - [a]_b */
  const uint64_t d = (d0 + d1) & M;                                 /* opened by P0 and P1 */
  const uint64_t e = (z - ((b0 + b1) & M)) & M;                     /* step 3: e = DReLU' - b */
  const uint64_t in0 = (d * e + d * b0 + e * a0 + c0) & M;          /* P0 adds de (C8) */
  const uint64_t in1 = (d * b1 + e * a1 + c1) & M;
  const uint64_t t = tp.t;
  *y0 = (t * x0 + (t ? (0ull - in0) : in0)) & M;                    /* step 5 */
  *y1 = (t * x1 + (t ? (0ull - in1) : in1)) & M;
}

/* ------------------------------------------------------------------------------------
 * Entry points.  Return 0, or -1 on bad parameters.  W0 / W1 (nullable): the messages,
 * n x S u64.  nthreads <= 0: OpenMP's default.
 * ---------------------------------------------------------------------------------- */
int bcref_version(void) { return 1; }

int bcref_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

int bcref_fused(int ell, int lx, int f, int literal, int rounds, const uint8_t *s01, const uint8_t *s02,
                const uint8_t *s12, const uint64_t *x0, const uint64_t *x1, uint64_t *y0, uint64_t *y1,
                uint64_t *W0, uint64_t *W1, int64_t n, uint64_t base, int relu, int nthreads) {
  prm_t P;
  if (prm_make(&P, ell, lx, f, literal, rounds)) return -1;
  if (nthreads <= 0) nthreads = bcref_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t w0[32], w1[32];
    one_element(&P, s01, s02, s12, x0[i], x1[i], base + (uint64_t)i, relu, &y0[i], &y1[i], w0, w1);
    if (W0) memcpy(W0 + (size_t)i * P.S, w0, sizeof(uint64_t) * P.S);
    if (W1) memcpy(W1 + (size_t)i * P.S, w1, sizeof(uint64_t) * P.S);
  }
  return 0;
}

/* Alg 7 steps 3-5 alone (config 2), one party, no blinding: v'_0 .. v'_lx per element. */
int bcref_ladder_modswitch(int ell, int lx, int f, int literal, int party, const uint64_t *x, uint64_t *vp, int64_t n,
                           int nthreads) {
  prm_t P;
  if (prm_make(&P, ell, lx, f, literal, 20) || (party != 0 && party != 1)) return -1;
  if (nthreads <= 0) nthreads = bcref_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
  for (int64_t i = 0; i < n; ++i) ladder_modswitch(&P, party, x[i], vp + (size_t)i * P.S);
  return 0;
}
