/*
 * bicoptor.h -- C ABI of libbicoptor: the B200 (sm_100a) hot path of the
 * Bicoptor 2.0 UBL DReLU / ReLU protocol (arXiv 2309.04909).
 *
 * Citations: "P:n" = line n of the paper's LaTeX source, with the
 * algorithm / section it falls in; readings Cn are listed in DESIGN.md.
 *
 * Conventions (every entry point)
 *   - Returns BC_OK (0) or a negative BC_E* code; bc_strerror() maps it to text.
 *   - All array arguments are DEVICE pointers owned by the caller.  The library
 *     never allocates, frees or synchronises; every call is asynchronous on
 *     `stream` (a cudaStream_t passed as void*, NULL = legacy default stream).
 *     Asynchronous CUDA faults surface at the caller's next synchronisation.
 *   - Share vectors are uint64_t[n]: element i holds a value of Z_{2^ell} in
 *     its low ell bits (high bits of inputs are ignored, high bits of outputs
 *     are zero).  Arrays of uint64_t must be 16-byte aligned (BC_EALIGN).
 *   - n = 0 is a no-op that still validates the parameters.
 *   - Inputs and outputs must not overlap (BC_EALIAS), except where stated.
 *   - elem_base is the global index of element 0 of this call; every PRG draw
 *     is addressed by global index j = elem_base + i, so a batch split into
 *     shards (or chunks) gives bit-identical results to one call.  It must be
 *     a multiple of 8 (BC_EALIGN), and elem_base + n <= BC_MAX_INDEX = 2^44
 *     (BC_ERANGE): the stream counters (j * 9 + b for the large tape, j * 2^20
 *     + k for its fallback stream) then never wrap.
 *   - Seeds are 32-byte keys passed by value; a party-phase call takes only the
 *     seeds that party holds: P0 {seed01, seed02}, P1 {seed01, seed12},
 *     P2 {seed02, seed12}.
 *   - Stateless and thread-safe.
 */
#ifndef BICOPTOR_H
#define BICOPTOR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BC_OK 0
#define BC_EINVAL (-1)   /* bad parameter (party id, ell, lx, mode, rounds, NULL) */
#define BC_ERANGE (-2)   /* key-bit window does not fit: need f + lx + w <= ell,
                            or elem_base + n > BC_MAX_INDEX                      */
#define BC_EALIGN (-3)   /* pointer not 16-B aligned, or elem_base % 8 != 0      */
#define BC_ECUDA  (-4)   /* CUDA launch error (bc_last_cuda_error() has the code) */
#define BC_EALIAS (-5)   /* an output overlaps an input                          */

#define BC_MAX_INDEX ((uint64_t)1 << 44) /* bound on global element indices (elem_base + n) */

#define BC_MODE_GUARD   0 /* w = lx + 1, p = 257 at lx = 7 (default; reading C6) */
#define BC_MODE_LITERAL 1 /* w = lx, the paper's Z_{2^lx} (64-bit wire)  */

/* PRG tape layouts. */
#define BC_TAPE_PAIR    0 /* lx <= 7, p <= 131 (other than the cases below): 32 B / element, 28-bit (r, rho) draws */
#define BC_TAPE_COMPACT 1 /* p = 257 and 8 slots (lx = 7 guard): 24 B / element            */
#define BC_TAPE_LARGE   2 /* lx >= 8, up to 32 slots and p < 2^33: 448 B / element          */
#define BC_TAPE_COMPACT_LIT 3 /* p = 131 and 8 slots (lx = 7 literal): the pair tape, kernels with constant parameters */

/* Protocol parameters (Alg 7 "Setting"; key bits, sec. 6.1).
 *   ell    ring bits, 2..64
 *   lx     ladder width ell_x, 2..31 (lx + 1 ladder slots).  lx = 7 is the
 *          paper's key-bit setting; lx = 31, f = 0 is its full 5+26
 *          precision without key bits
 *   f      window offset: the ladder reads bits [f, f+lx+w) (reading C5;
 *          f = 24 keeps 5+2 of the paper's 5+26 fixed point)
 *   mode   BC_MODE_GUARD / BC_MODE_LITERAL
 *   rounds ChaCha rounds 8, 12 or 20 (reading C19)
 * Derived by bc_params_init: w (window width), p (smallest prime > 2^w,
 * reading C7; 2^32 + 15 at lx = 31 guard), slots = lx + 1, tape (BC_TAPE_*).
 * bc_ladder_modswitch (a byte-plane format) needs slots <= 8 and p <= 257
 * (BC_EINVAL otherwise); the party phases use byte planes for those and
 * uint32 planes for the large tape (bc_drelu_send); bc_drelu / bc_relu accept
 * every tape. */
typedef struct bc_params {
  int32_t ell, lx, f, mode, rounds;
  uint32_t w, slots;
  int32_t tape;
  uint64_t p;
} bc_params;

/* Pre-shared seeds seed01, seed02, seed12. */
typedef struct bc_seeds {
  uint8_t s01[32];
  uint8_t s02[32];
  uint8_t s12[32];
} bc_seeds;

/* Optional transcript of the simulated three-party run (bc_drelu / bc_relu):
 * the messages P0 and P1 send to P2 (Alg 7 step 8).  Compact and pair
 * tapes: the wire format of bc_drelu_send, all four planes non-NULL.  Large
 * tape: w0_lo and w1_lo are uint64_t[n][slots] (W_m in [0, p), 8-B aligned),
 * w0_hi and w1_hi must be NULL. */
typedef struct bc_transcript {
  uint8_t *w0_lo, *w0_hi, *w1_lo, *w1_hi;
} bc_transcript;

/* Validate and derive parameters.  BC_EINVAL / BC_ERANGE on bad input. */
int bc_params_init(bc_params *out, int ell, int lx, int f, int mode, int rounds);

/* Alg 4 / Alg 5 deterministic truncation for one party:
 *   P0: out = cut(in, k1, k2) mod 2^(ell-k1-k2)
 *   P1: out = 2^ell - cut(2^ell - in, k1, k2) mod 2^(ell-k1-k2)  (readings C2-C4)
 * k2 = 0 is Alg 4.  Requires k1 + k2 < ell.  in, out: uint64_t[n]. */
int bc_trc(int party, const uint64_t *in, uint64_t *out, size_t n, int ell, int k1, int k2,
           void *stream);

/* Alg 1 SecureML probabilistic truncation for one party, the
 * prior-work baseline whose e1 error the paper analyses:
 *   P0: cut(in, k) mod 2^ell;  P1: 2^ell - cut(2^ell - in, k) mod 2^ell (C3). */
int bc_trc_prob(int party, const uint64_t *in, uint64_t *out, size_t n, int ell, int k,
                void *stream);

/* Alg 6 modulo switch for one party: shares of x in Z_{2^lp} ->
 * shares in Z_p.  P0: in == 0 ? 2^lp mod p : in mod p;  P1: (p + in - 2^lp) mod p.
 * Requires 1 <= lp <= 31 and 2^lp < p < 2^32 (p need not be checked prime).
 * in: uint64_t[n] (low lp bits used), out: uint32_t[n] (4-B aligned). */
int bc_modswitch(int party, const uint64_t *in, uint32_t *out, size_t n, int lp, uint32_t p,
                 void *stream);

/* Alg 7 steps 3-5 for one party on its share as given (no blinding bit, no
 * shuffle): ladder u_i = Alg 5 with k1 = f+i, k2 = ell-w-f-i,
 * pairwise v_i (P0 carries the -1, reading C8), modulo switch
 * (Alg 6).  Output v: uint8_t[n][8], byte m of row i = v'_m - 1 (v' lies in
 * Z_p^* so this is lossless for p <= 257), bytes m >= slots are 0.  v must be
 * 16-B aligned. */
int bc_ladder_modswitch(int party, const uint64_t *x, uint8_t *v, size_t n,
                        const bc_params *prm, void *stream);

/* Alg 6 at any width, for the full-precision guard domain (lp = 32,
 * p = 2^32 + 15) and beyond: shares in Z_{2^lp} -> shares in Z_p, as
 * bc_modswitch.  Requires 1 <= lp <= 63 and 2^lp < p (p < 2^64; p need not be
 * checked prime).  in: uint64_t[n] (low lp bits used), out: uint64_t[n]; both
 * 16-B aligned, caller-owned, not overlapping.  Both results already lie in
 * [0, p): P0's share is in (0, 2^lp], P1's in [p - 2^lp, p). */
int bc_modswitch64(int party, const uint64_t *in, uint64_t *out, size_t n, int lp, uint64_t p,
                   void *stream);

/* Alg 7 steps 3-5 for one party, every tape including the large one (lx up to
 * 31, p < 2^33; Alg 5, Alg 6): as
 * bc_ladder_modswitch, but the output is the v'_m themselves, uint64_t[n][slots]
 * (row-major, slot m of element i at v[i * slots + m]), each in [1, p).  x and v
 * 16-B aligned, caller-owned, not overlapping. */
int bc_ladder_modswitch64(int party, const uint64_t *x, uint64_t *v, size_t n,
                          const bc_params *prm, void *stream);

/* Alg 7, all three parties simulated on one GPU in one fused
 * kernel: y0 + y1 = DReLU(x0 + x1) mod 2^ell (1 for positive, 0 for negative
 * in-band x; x = 0 gives the random bit t, reading C13).  tr may be NULL.
 * Without a transcript P2 tests P0's reduced message against P1's congruent
 * integer; the environment variable BICOPTOR_MATERIALIZE=2,
 * read on each call, selects an instantiation that reduces both messages to
 * wire values first (a measurement knob: the outputs are identical). */
int bc_drelu(const uint64_t *x0, const uint64_t *x1, uint64_t *y0, uint64_t *y1, size_t n,
             uint64_t elem_base, const bc_params *prm, const bc_seeds *seeds,
             const bc_transcript *tr, void *stream);

/* Alg 8, all three parties on one GPU in one fused kernel:
 * y0 + y1 = x * DReLU(x) mod 2^ell (x = x0 + x1). */
int bc_relu(const uint64_t *x0, const uint64_t *x1, uint64_t *y0, uint64_t *y1, size_t n,
            uint64_t elem_base, const bc_params *prm, const bc_seeds *seeds,
            const bc_transcript *tr, void *stream);

/* Bicoptor-1 DReLU as Bicoptor 2.0 describes its predecessor -- an in-repo
 * comparison point (readings C32-C34): SecureML truncation
 * (u_i in Z_{2^ell}, probabilistic), recursive sums, no modulo
 * switch, odd masks and reshares in Z_{2^ell}; (lx+1) * ell message bits per
 * party.  Arguments as bc_drelu; prm->slots <= 8; tr, if given,
 * receives W0, W1 as uint64_t[n][slots] planes in w0_lo / w1_lo (hi NULL). */
int bc_drelu_b1(const uint64_t *x0, const uint64_t *x1, uint64_t *y0, uint64_t *y1, size_t n,
                uint64_t elem_base, const bc_params *prm, const bc_seeds *seeds,
                const bc_transcript *tr, void *stream);

/* ---- host-buffer entry points (end to end) ------------------------------
 *
 * bc_drelu / bc_relu on shares that live in HOST memory: x0, x1 (in) and y0,
 * y1 (out) are host arrays of n uint64_t (pinned memory recommended; pageable
 * works but serialises the copies).  The batch is processed in chunks of
 * `chunk` elements (a positive multiple of 8): H2D copy, the fused kernel
 * (elem_base + chunk offset, so the result equals one bc_drelu over the whole
 * batch), D2H copy, pipelined over a ring of 3 library-owned CUDA streams so
 * both PCIe directions overlap each other and the kernels.  ws is a caller-
 * owned DEVICE workspace of ws_bytes >= bc_host_workspace_bytes(chunk), 16-B
 * aligned.  Ordered after prior work on `stream`; unlike every other entry
 * point the call is synchronous: the host outputs are complete on return.
 * Errors as bc_drelu (BC_EINVAL for a short workspace or a bad chunk). */
size_t bc_host_workspace_bytes(size_t chunk);
int bc_drelu_host(const uint64_t *x0, const uint64_t *x1, uint64_t *y0, uint64_t *y1, size_t n,
                  uint64_t elem_base, const bc_params *prm, const bc_seeds *seeds, void *ws,
                  size_t ws_bytes, size_t chunk, void *stream);
int bc_relu_host(const uint64_t *x0, const uint64_t *x1, uint64_t *y0, uint64_t *y1, size_t n,
                 uint64_t elem_base, const bc_params *prm, const bc_seeds *seeds, void *ws,
                 size_t ws_bytes, size_t chunk, void *stream);

/* Asynchronous forms of the two calls above: enqueue only.  The chunks are not
 * ordered after the caller's earlier stream work (the host inputs must be
 * ready when called); the caller's stream waits for every chunk, so
 * synchronising it makes the host outputs complete.  Consecutive calls with
 * the same workspace pipeline into each other: a serving loop keeps both PCIe
 * directions busy across requests instead of filling and draining per call.
 * The host buffers of a call must not be reused before that point. */
int bc_drelu_host_async(const uint64_t *x0, const uint64_t *x1, uint64_t *y0, uint64_t *y1,
                        size_t n, uint64_t elem_base, const bc_params *prm,
                        const bc_seeds *seeds, void *ws, size_t ws_bytes, size_t chunk,
                        void *stream);
int bc_relu_host_async(const uint64_t *x0, const uint64_t *x1, uint64_t *y0, uint64_t *y1,
                       size_t n, uint64_t elem_base, const bc_params *prm, const bc_seeds *seeds,
                       void *ws, size_t ws_bytes, size_t chunk, void *stream);

/* ---- party-separated phases (each party on its own device; the caller moves
 * the message buffers, e.g. with NCCL send/recv) --------------------------- */

/* Alg 7 steps 1-8 for P0 (party 0) or P1 (party 1): the message to P2 in the
 * wire format lo: uint8_t[n][8] (low 8 bits of W_m, 16-B aligned), hi:
 * uint8_t[n] (bit m = bit 8 of W_m; may be NULL when p <= 256), plus the
 * party's blinding bits tbits: uint8_t[(n+7)/8] (bit i%8 of byte i/8 = t_i),
 * kept locally for the finish phase.  (lx+1)*ceil(log2 p) bits per element:
 * 72 in guard mode, 64 literal (Table 1).
 * Large tape (lx >= 8, S = lx+1 <= 32 slots, p < 2^33): lo is the
 * slot-major plane uint32_t[S][n] (lo[m n + i] = low 32 bits of element i's
 * W_m, so a warp's stores and loads of one slot are contiguous) and hi is
 * uint32_t[n] (bit m = bit 32 of W_m; may be NULL when p < 2^32): 33 S bits
 * per element, 1,056 at the full precision lx = 31 (the paper's "31 * 31 ~
 * 1,000 bits").  The helper (bc_drelu_helper, bc_relu_helper[_to])
 * takes the same planes. */
int bc_drelu_send(int party, const uint64_t *x, uint8_t *lo, uint8_t *hi, uint8_t *tbits,
                  size_t n, uint64_t elem_base, const bc_params *prm, const uint8_t seed01[32],
                  void *stream);

/* P0's whole DReLU in the transport where P0 derives [D']_0 from seed02 itself
 * (reading C12; P2 answers only P1): Alg 7 steps 1-8 as bc_drelu_send for
 * party 0, and steps 10-11 in the same kernel, y[i] = t + (1-2t) q with q the
 * seed02 response stream (the value bc_drelu_finish would compute).  y:
 * uint64_t[n], 16-B aligned; tbits may be NULL (it is not needed afterwards).
 * BC_EINVAL for y == NULL or seed02 == NULL. */
int bc_drelu_send_p0(const uint64_t *x, uint8_t *lo, uint8_t *hi, uint8_t *tbits, uint64_t *y,
                     size_t n, uint64_t elem_base, const bc_params *prm, const uint8_t seed01[32],
                     const uint8_t seed02[32], void *stream);

/* Alg 7 steps 9-10 for P2: zero test of w = W0 + W1 mod p, then
 * reshare DReLU' in Z_{2^ell}: [D']_0 = seed02 stream value (P0 can derive
 * it; written to resp0 only if resp0 != NULL, the paper-literal transport,
 * reading C12), resp1 = DReLU' - [D']_0.  resp0/resp1: uint64_t[n]. */
int bc_drelu_helper(const uint8_t *lo0, const uint8_t *hi0, const uint8_t *lo1,
                    const uint8_t *hi1, uint64_t *resp0, uint64_t *resp1, size_t n,
                    uint64_t elem_base, const bc_params *prm, const uint8_t seed02[32],
                    void *stream);

/* Alg 7 step 11: y = t + (1-2t)[D']_b (P0 adds t, reading C8).
 * P0 with resp == NULL derives [D']_0 from seed02 itself (pass seed02; P1
 * passes NULL). */
int bc_drelu_finish(int party, const uint8_t *tbits, const uint64_t *resp, uint64_t *y,
                    size_t n, uint64_t elem_base, const bc_params *prm,
                    const uint8_t seed02[32], void *stream);

/* Alg 8 step 1 and the first half of step 4 for P0 / P1: the Alg 7 message
 * (as bc_drelu_send) and the party's share of d = x - a: dshare = x_b - [a]_b,
 * sent to the other computing party.  seed_tr = seed02 for P0, seed12 for P1
 * (Alg 8 preprocessing). */
int bc_relu_send(int party, const uint64_t *x, uint8_t *lo, uint8_t *hi, uint8_t *tbits,
                 uint64_t *dshare, size_t n, uint64_t elem_base, const bc_params *prm,
                 const uint8_t seed01[32], const uint8_t seed_tr[32], void *stream);

/* Alg 8 steps 2-3 for P2: DReLU' by the zero test, e = DReLU' -
 * ([b]_0 + [b]_1) sent to both, and [c]_1 = ([a]_0+[a]_1)([b]_0+[b]_1) - [c]_0
 * sent to P1 (c1 may be NULL if it was delivered in preprocessing, C20). */
int bc_relu_helper(const uint8_t *lo0, const uint8_t *hi0, const uint8_t *lo1,
                   const uint8_t *hi1, uint64_t *e, uint64_t *c1, size_t n, uint64_t elem_base,
                   const bc_params *prm, const uint8_t seed02[32], const uint8_t seed12[32],
                   void *stream);

/* Alg 8 steps 4-5 for P0 / P1: d = d_own + d_peer, then
 * y_b = t x_b + (1-2t)(de + d[b]_b + e[a]_b + [c]_b), P0 adding de (C8).
 * c1 is P1's [c]_1 (NULL for P0).  seed_tr as in bc_relu_send. */
int bc_relu_finish(int party, const uint64_t *x, const uint8_t *tbits, const uint64_t *d_own,
                   const uint64_t *d_peer, const uint64_t *e, const uint64_t *c1, uint64_t *y,
                   size_t n, uint64_t elem_base, const bc_params *prm,
                   const uint8_t seed_tr[32], void *stream);

/* Peer-memory variants of the ReLU phases (the transport of
 * paper_2309_04909_b200/peer.py).  As bc_relu_send, and
 * [d]_b is stored a second time into dshare_peer (nullable): a device pointer
 * that may be the other computing party's receive buffer mapped into this
 * process by bc_ipc_open (on another GPU: a peer mapping, the stores travel
 * over NVLink).  dshare_peer must be 16-B aligned and must not overlap x or
 * dshare (BC_EALIAS is checked in this process's address space only). */
int bc_relu_send_to(int party, const uint64_t *x, uint8_t *lo, uint8_t *hi, uint8_t *tbits,
                    uint64_t *dshare, uint64_t *dshare_peer, size_t n, uint64_t elem_base,
                    const bc_params *prm, const uint8_t seed01[32], const uint8_t seed_tr[32],
                    void *stream);

/* As bc_relu_helper, with e stored to e0 (P0's copy) and, if e1 != NULL, a
 * second time to e1 (P1's copy): Alg 8 step 3 sends e to both computing
 * parties.  e1 != NULL requires e0 != NULL (BC_EINVAL). */
int bc_relu_helper_to(const uint8_t *lo0, const uint8_t *hi0, const uint8_t *lo1,
                      const uint8_t *hi1, uint64_t *e0, uint64_t *e1, uint64_t *c1, size_t n,
                      uint64_t elem_base, const bc_params *prm, const uint8_t seed02[32],
                      const uint8_t seed12[32], void *stream);

/* ---- peer memory (CUDA IPC) -------------------------------------------------
 * Host-only plumbing for the peer-memory transport; no kernel is launched.
 * bc_ipc_export: handle (64 B, caller-owned host memory) of the device
 * allocation that contains dptr, and dptr's byte offset inside it (allocators
 * sub-allocate, so the handle names the whole allocation).  bc_ipc_open maps
 * a handle exported by ANOTHER process into this one (*base = the mapping of
 * the allocation's first byte; peer access is enabled lazily when the
 * allocation lives on another GPU); bc_ipc_close unmaps it.  The exporter
 * keeps the allocation alive until every importer has closed it.  Errors:
 * BC_EINVAL for NULL arguments, BC_ECUDA otherwise (bc_last_cuda_error). */
int bc_ipc_export(const void *dptr, uint8_t handle[64], uint64_t *offset);
int bc_ipc_open(const uint8_t handle[64], void **base);
int bc_ipc_close(void *base);

/* ---- RSS variant (Alg 9; RSS ReLU P:1930-1931) -------------
 *
 * Replicated 3-party sharing x = x0 + x1 + x2 mod 2^ell (P_i holds
 * components i and i+1).  All three parties simulated in one fused kernel:
 * the preprocessing ([t] re-shared from seed012, [s], [u] = [s XOR t] by one
 * RSS multiplication), Alg 7 on the bridged sharing (P0 input x0 + x1, P1
 * input x2; Alg 9 online step 1), DReLU'' = s XOR DReLU' (step 3) and the
 * output [DReLU] = DReLU'' + [u] - 2 DReLU''[u] (step 5; DReLU'' on component
 * 0, reading C27).  bc_relu_rss adds the secret multiplication [x][DReLU]
 * (reading C26: z_i = a_i b_i + a_i b_{i+1} + a_{i+1} b_i + g_i, g a zero
 * sharing from seed02 / seed01 / seed12).  Stream labels: DESIGN.md C25.
 *
 * x0, x1, x2 (in) and y0, y1, y2 (out): n u64 components in [0, 2^ell),
 * device memory, 16-B aligned, outputs disjoint from each other and from the
 * inputs (BC_EALIAS).  seeds: the pairwise seeds; seed012: the seed of all
 * three parties; seed2: P2's private seed (32 B each, host memory).  Only the
 * compact tape (guard mode, p = 257) is supported (BC_EINVAL otherwise).
 * Errors as bc_drelu; elem_base % 8 == 0; n = 0 is a no-op. */
int bc_drelu_rss(const uint64_t *x0, const uint64_t *x1, const uint64_t *x2, uint64_t *y0,
                 uint64_t *y1, uint64_t *y2, size_t n, uint64_t elem_base, const bc_params *prm,
                 const bc_seeds *seeds, const uint8_t seed012[32], const uint8_t seed2[32],
                 void *stream);

/* RSS ReLU: [x][DReLU(x)]; arguments as bc_drelu_rss. */
int bc_relu_rss(const uint64_t *x0, const uint64_t *x1, const uint64_t *x2, uint64_t *y0,
                uint64_t *y1, uint64_t *y2, size_t n, uint64_t elem_base, const bc_params *prm,
                const bc_seeds *seeds, const uint8_t seed012[32], const uint8_t seed2[32],
                void *stream);

/* ---- truncation study (sec. 3-5) --------------------
 *
 * Probabilistic truncation of prior work and its error e1 (sec. 4),
 * the deterministic Alg 4 for comparison, and Alg 3 "truncate-then-multiply"
 * (sec. 5.2).  Two parties simulated on one GPU; the preprocessing
 * comes from the seeds with P2 as the dealer (readings C29, C31). */
#define BC_TRC_SECUREML 1 /* Alg 1, non-interactive probabilistic */
#define BC_TRC_ABY3     2 /* Alg 2, interactive probabilistic      */
#define BC_TRC_DET      4 /* Alg 4, deterministic, Z_{2^(ell-k)}   */
#define BC_MUL_THEN_TRC 0 /* z = x y, then trc(z, f)                           */
#define BC_TRC_THEN_MUL 1 /* Alg 3: trc(x, floor(f/2)) trc(y, ceil(f/2))        */

/* Alg 2 (ABY3) for both parties: alpha = x + r is opened ([x]_i + [r]_i, the
 * paper's footnote P:341), y0 = alpha/2^k - [r']_0 (P0 adds the public term,
 * C29), y1 = -[r']_1.  r, r' = cut(r, k) preprocessed from seed02 / seed12,
 * truncation instance q (0 or 1) selecting the labels.  y0 + y1 = trc(x, k) up
 * to e0, or e1 when x + r wraps.  Arrays as bc_drelu; 2 <= ell <= 64,
 * 0 <= k < ell, rounds 8 / 12 / 20. */
int bc_trc_aby3(const uint64_t *x0, const uint64_t *x1, uint64_t *y0, uint64_t *y1, size_t n,
                uint64_t elem_base, int ell, int k, int rounds, int q, const bc_seeds *seeds,
                void *stream);

/* Exact e1 counting (sec. 4).  For each plaintext x[i] (i < nx; device
 * uint64_t, 8-B aligned) and each mask m in [m_base, m_base + m_count) (taken
 * mod 2^ell), run alg on the shares -- Alg 1 / Alg 4: [x]_0 = x + m, [x]_1 = -m;
 * Alg 2: r = m -- and add the class of the reconstruction (reading C30:
 * exact, e0 = the one-bit error, e1 = anything else) to counts[i][0..2]
 * (uint64_t[nx][3], accumulated: the caller zeroes it).  Over all 2^ell masks
 * Alg 1 / Alg 2 give e1 = xi for every x (C18); Alg 4 gives none (Theorem
 * newcut2).  1 <= k < ell <= 64. */
int bc_trc_count(int alg, const uint64_t *x, size_t nx, int ell, int k, uint64_t m_base,
                 uint64_t m_count, uint64_t *counts, void *stream);

/* Secure fixed-point multiplication z = x y / 2^f for both parties (a Beaver
 * product, triple from seed02 / seed12 by P2, C31), in the order given:
 * BC_MUL_THEN_TRC (truncate the product) or BC_TRC_THEN_MUL (Alg 3: truncate
 * the operands by floor(f/2) and ceil(f/2), then multiply), each truncation
 * Alg 1 or Alg 2 (alg).  Arrays as bc_drelu; 0 <= f < ell. */
int bc_mul_trc(int order, int alg, const uint64_t *x0, const uint64_t *x1, const uint64_t *y0,
               const uint64_t *y1, uint64_t *z0, uint64_t *z1, size_t n, uint64_t elem_base,
               int ell, int f, int rounds, const bc_seeds *seeds, void *stream);

/* Human-readable text for a BC_* code (static storage). */
const char *bc_strerror(int code);

/* cudaError_t of the most recent BC_ECUDA on this thread (0 if none). */
int bc_last_cuda_error(void);

/* Library ABI version (major * 100 + minor).  3.00: the large-tape party
 * phases (slot-major uint32 wire planes), bc_relu_send_to / bc_relu_helper_to,
 * bc_ipc_*, BC_MAX_INDEX, and the 7-block large tape bc2.tpL2 (2.00: 9 blocks).
 * 3.01: the 32-B pair tape bc2.tpp1 (BC_TAPE_PAIR, BC_TAPE_COMPACT_LIT) replaces the
 * 64-B wide tape: every lx <= 7 domain but the compact one draws different keystream. */
int bc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BICOPTOR_H */
