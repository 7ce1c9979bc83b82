/*
 * gb.h -- C-ABI of libgb: batched retrieval in the Gripon-Berrou clustered
 * associative memory (GBNN), arXiv:1303.7032, on NVIDIA B200 (sm_100a).
 *
 * The paper's problem statement has two operations, storing and retrieving
 * (PAPER.md L35-37).  This header exposes exactly those, plus the handle
 * lifecycle and the plumbing a multi-GPU caller needs (W exposure for an
 * NCCL broadcast / MAX all-reduce).
 *
 * Conventions:
 *  - 0-based clusters, neurons and symbols (reading R1).  A message or probe
 *    is uint16_t[C]; symbol in [0, L), GB_ERASED (0xFFFF) marks an erased
 *    cluster of a probe ("(m_1, m_2, ?, ?)").
 *  - Cluster padding: each cluster occupies Wc = ceil(L/32) 32-bit words,
 *    Lp = 32*Wc neuron slots; n_padded = C*Lp.  Neuron (c, l) has padded
 *    index i = c*Lp + l (the paper's i = (c-1)L + l of L310 with padding).
 *    Padding neurons never activate and have no edges.
 *  - A decoded state is uint32_t[C*Wc]: bit (l % 32) of word c*Wc + l/32 is
 *    v_(c,l); padding bits are 0.
 *  - Every pointer argument is a plain pointer.  For gb_store and gb_decode
 *    buffers may be device pointers (on the handle's device) or host
 *    pointers (pageable or pinned); host buffers are staged through the
 *    library's device scratch (gb_decode*: chunks of 2^19 probes pipelined
 *    through three slots on a copy-in, a compute and a copy-out stream, so
 *    both PCIe directions stay busy) and the call then blocks until the
 *    results are back in host memory.  Device-pointer calls are asynchronous and
 *    stream-ordered on `stream` (a cudaStream_t, NULL = legacy default).
 *  - The caller owns all input/output buffers.  The library owns W (u8 and
 *    bit-packed), its sum-of-sum operands W8 + gamma*I, and a memory pool.
 *  - Concurrency.  After gb_seal, W is
 *    immutable and any number of host threads may call gb_decode /
 *    gb_decode_ex on one handle at the same time, on any streams, with any
 *    rules and gammas, provided their output buffers are distinct: every
 *    decode allocates its scratch (work counters, overflow lists, state
 *    scratch) stream-ordered from the handle's pool, so no two calls share a
 *    device buffer the kernels write.  Calls that change W (gb_clear,
 *    gb_store, gb_or_bits, gb_or_upper, gb_seal, writes through gb_weights' pointer) and
 *    gb_set_option must not overlap decodes on the handle and must be ordered
 *    with them (same stream, or events).  Host-buffer calls (see above) of one
 *    handle are serialised internally.  Results do not depend on how a batch
 *    is split over calls or streams (Eq.(11): independent columns).
 *  - Errors: functions return GB_OK (0) or a negative GB_E* code and set a
 *    thread-local message readable with gb_last_error().  No exception or
 *    abort crosses the ABI.  There is no CPU fallback: without a usable
 *    sm_100 device every compute call fails with GB_ECUDA/GB_EUNSUPPORTED.
 */
#ifndef GB_H
#define GB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gb_net gb_net;

enum {
    GB_OK = 0,
    GB_EINVAL = -1,        /* bad argument or invalid symbol (see each call) */
    GB_ENOMEM = -2,        /* device allocation failed                       */
    GB_ECUDA = -3,         /* CUDA runtime error (message has the details)   */
    GB_ESTATE = -4,        /* call not allowed in the handle's state         */
    GB_EUNSUPPORTED = -5   /* shape or device outside what libgb supports    */
};

/* Retrieval rules. */
enum {
    GB_SUM_OF_SUM = 0,     /* Eq.(3)-(5), Alg. 1 */
    GB_SUM_OF_MAX = 1,     /* Eq.(6)-(7) via bail-out-early (L258-265, L439-483) */
    GB_HYBRID = 2          /* joint scheme, Alg. 2 (L596-683)                   */
};

/* Per-probe status written by gb_decode. */
enum {
    GB_CONVERGED = 0,      /* V^r == V^{r-1} for some round r <= max_iters     */
    GB_MAX_ITERS = 1,      /* max_iters rounds ran without a fixed point        */
    GB_INVALID = 2,        /* a probe symbol was >= L (and not GB_ERASED); the
                              state is all zero and iters is 0                  */
    GB_CYCLE = 3           /* only with GB_FLAG_CYCLE_EXIT: sum-of-sum state of
                              round r repeats round r-2 (period-2 oscillation)  */
};

/* Kernel-selection options (gb_set_option).  They choose between kernels
 * that compute the same results (bit-exact); the defaults are the measured
 * fastest.  No environment variable or other global state is read. */
enum {
    GB_OPT_SOS_PAIR = 0,       /* 1 (default): sum-of-sum on CTA pairs (cta_group::2)
                                  where the shape allows; 0: one CTA per tile       */
    GB_OPT_SOS_STREAMED = 1,   /* 1 (default): streamed-A sum-of-sum kernel for
                                  1024 < n_padded <= 4096; 0: the 4-warp kernel      */
    GB_OPT_SOM_TENSOR = 2,     /* 1: sum-of-max as exact int8 contractions on the
                                  tensor cores (n_padded <= 1024);
                                  0 (default): the bit-row kernels                   */
    GB_OPT_HYB8 = 3,           /* 1 (default): the C = 8 hybrid kernel; 0: the
                                  general shared-memory hybrid kernel               */
    GB_OPT_L2T = 4,            /* 1 (default): thread-per-probe L2 bit kernel; 0:
                                  warp-per-probe kernel (W rows beyond shared mem)   */
    GB_OPT_HYB8_SPLIT = 5,     /* -1 (default): choose the C = 8 hybrid kernel by
                                  W's density (known once a seal's status reached
                                  the host): the rotated-layout kernel when dense
                                  (>0.65), the uniform-loop kernel when sparse;
                                  0 (loop) / 1 (rotated) force it (bit-exact)        */
    GB_OPT_STORE_SCATTER = 6,  /* 1: gb_store with scattered byte writes only;
                                  0 (default): shared-memory privatised tiles for
                                  large batches                                      */
    GB_OPT_HYB8_ROWS = 7,      /* 0 (default): rows of the rotated-layout hybrid
                                  kernel's first push step chosen by W's density;
                                  6..8 force it (bit-exact either way)               */
    GB_OPT_SOS_BITS = 8        /* -1 (default): sum-of-sum on the CUDA cores (the
                                  active rows into bit-sliced counters) when W is
                                  sparse (density < 0.45; C <= 8, n_padded <= 1024,
                                  no cycle exit), else on the tensor cores; 0 / 1
                                  force it (bit-exact either way)                    */
};

/* gb_decode_ex flags. */
enum {
    GB_FLAG_CYCLE_EXIT = 1 /* sum-of-sum: stop a probe at the first round r >= 2
                              with V^r == V^{r-2} != V^{r-1} (the period-2
                              oscillation of PAPER.md L515-522) with status
                              GB_CYCLE, iters r and state V^r, instead of running
                              to max_iters.  SURVEY.md §8.f N4 / SPEC S:L304.
                              Changes the returned state (V^r, not V^max_iters),
                              so it is off by default.  No effect on sum-of-max
                              and hybrid, whose rounds only remove neurons
                              (Lemma 1) and cannot oscillate.                     */
};

#define GB_ERASED 0xFFFFu
#define GB_AMBIGUOUS 0xFFFEu   /* gb_decode_symbols: several neurons of a cluster active */

/*
 * gb_create -- a network of c clusters with l neurons each (PAPER.md L144-145,
 * "n = CL binary-valued neurons ... grouped into C clusters of L neurons"),
 * all edges zero (L149), on CUDA device `device`.
 *   c in [2, 64], l >= 1, n_padded = c*32*ceil(l/32) <= 8192.
 *   Returns GB_EINVAL for c < 2 or l < 1, GB_EUNSUPPORTED beyond the limits
 *   or when `device` is not an sm_100 (B200-class) GPU, GB_ENOMEM if W does
 *   not fit.  *out receives the handle.
 */
int gb_create(int c, int l, int device, gb_net **out);

/* gb_destroy -- release W and scratch.  Synchronizes the device.  NULL ok. */
int gb_destroy(gb_net *net);

/*
 * gb_clear -- reset W to the empty network (all w_ij = 0) and
 * the stored count to 0; unseals.  Stream-ordered.
 */
int gb_clear(gb_net *net, void *stream);

/*
 * gb_store -- OR the clique of each of the m messages into W (PAPER.md
 * L149-153: "we add edges to the network connecting all pairs of nodes
 * which are activated"; Eq.(1)): for every message and every
 * cluster pair c != c', w_{(c,m_c)(c',m_c')} = w_{(c',m_c')(c,m_c)} = 1.
 * msgs: uint16_t[m][c], row-major.  OR is idempotent and commutative, so
 * calls may come in any order and from any stream split.
 * A message holding a symbol >= l (GB_ERASED included) stores nothing and
 * is counted on the device; the count is reported by gb_seal_status.
 * Unseals the network.  m == 0 is a no-op.  Returns GB_EINVAL for m < 0 or
 * NULL msgs with m > 0.
 */
int gb_store(gb_net *net, const uint16_t *msgs, int64_t m, void *stream);

/*
 * gb_set_option / gb_get_option -- per-handle kernel selection (GB_OPT_*).
 * value is 0 or 1 (GB_OPT_HYB8_SPLIT and GB_OPT_SOS_BITS also -1;
 * GB_OPT_HYB8_ROWS 0 or 6..8).
 * GB_EINVAL for an unknown
 * option or value.  Not to be called while decodes on the handle run.
 */
int gb_set_option(gb_net *net, int option, int value);
int gb_get_option(gb_net *net, int option, int *value);

/*
 * gb_weights -- expose the library-owned u8 weight matrix W8
 * (n_padded x n_padded, row-major, W8[i][j] = w_ij in {0,1}, diagonal 0;
 * gamma is applied at decode, reading R2).  Used for NCCL
 * broadcast (replicate W) and all-reduce MAX on uint8 (merge sharded
 * stores: max over {0,1} is OR).  Handing out the writable pointer (w8 not
 * NULL) unseals the network: decode returns GB_ESTATE until the next
 * gb_seal, so a W8 edit can never be decoded through a stale packed copy.
 * *w8 is a device pointer.  w8 == NULL only reports the size.
 */
int gb_weights(gb_net *net, uint8_t **w8, int64_t *nbytes);

/*
 * gb_weights_view -- the same W8 pointer for reading only (an NCCL broadcast
 * source, a comparison): the net stays sealed.  Writing through it is a
 * contract violation (decode would keep using the packed copy); use
 * gb_weights to edit W8.
 */
int gb_weights_view(gb_net *net, const uint8_t **w8, int64_t *nbytes);

/*
 * gb_bits -- expose the library-owned packed rows Wb (n_padded x n_padded/32
 * uint32, bit b of word w of row i = w_{i,32w+b}), valid after a successful
 * gb_seal and until the next gb_store / gb_clear / gb_or_bits / W8 edit.
 * This is the compact form for merging sharded stores:
 * all-gather the ranks' Wb (8x fewer bytes than the u8 W8) and OR them in
 * with gb_or_bits.  *wb is a device pointer.  Returns GB_ESTATE if unsealed.
 */
int gb_bits(gb_net *net, uint32_t **wb, int64_t *nbytes);

/*
 * gb_or_bits -- OR `count` packed bit matrices (device pointer to count
 * consecutive n_padded x n_padded/32 uint32 matrices in the gb_bits layout)
 * into W8: w_ij |= bit (i, j) of any of them.  Eq.(1) is an OR of cliques
 * (PAPER.md L149-153), so OR-ing the partial W's of message shards gives the
 * W of the whole message set.  Unseals; stream-ordered.  count == 0 is a
 * no-op; GB_EINVAL for count < 0 or NULL bits.  A matrix that breaks Eq.(1)'s
 * structure (asymmetric, intra-cluster or padding bits) is reported by the
 * next gb_seal.
 */
int gb_or_bits(gb_net *net, const uint32_t *bits, int64_t count, void *stream);

/*
 * gb_or_bits_multimem -- the NVLS form of gb_or_bits:
 * mc_bits is a MULTICAST address (a multicast object, e.g. torch symmetric
 * memory's multicast_ptr, mapped over one n_padded x n_padded/32 uint32
 * buffer per participating GPU, every rank's partial Wb at the same offset).
 * One multimem.ld_reduce.or per word reads the OR over all GPUs' copies,
 * reduced inside the NVSwitch, and sets those bits in W8 (w_ij |= ...).
 * Every rank must have written its copy before the call (a barrier over the
 * group); the caller keeps the buffers unchanged until the kernel is done.
 * Unseals; stream-ordered.  GB_EINVAL for NULL or misaligned mc_bits; a
 * non-multicast address fails at launch (GB_ECUDA).  Eq.(1) is an OR of
 * cliques, so the result is the W of all shards.
 */
int gb_or_bits_multimem(gb_net *net, const uint32_t *mc_bits, void *stream);

/*
 * gb_pack_upper -- the upper triangle of the sealed Wb, packed: for every
 * cluster pair a < b (lexicographic), the Lp x Wc words of Wb rows
 * a*Lp .. a*Lp+Lp-1, words b*Wc .. b*Wc+Wc-1, row-major.  W is symmetric
 * (PAPER.md L306), so this carries all of W in C(C-1)/2 of the C^2 blocks:
 * the smallest form to exchange between ranks (about
 * half of gb_bits' bytes).  *nwords (if not NULL) receives the uint32 count
 * (Lp*Wc*C*(C-1)/2); out may be NULL to query it, else a device buffer of
 * that many words on the handle's device.  Stream-ordered.  GB_ESTATE if not
 * sealed.
 */
int gb_pack_upper(gb_net *net, uint32_t *out, int64_t *nwords, void *stream);

/*
 * gb_or_upper -- OR `count` packed upper-triangle sets (consecutive, each in
 * gb_pack_upper's layout, device memory) into W8, both w_ij and its mirror
 * w_ji (Eq.(1) stores both directions).  Unseals; stream-ordered; count == 0
 * is a no-op; GB_EINVAL for count < 0 or NULL sets.
 */
int gb_or_upper(gb_net *net, const uint32_t *sets, int64_t count, void *stream);

/*
 * gb_seal -- freeze W for retrieval ("At the retrieval stage,
 * the variables w are fixed"): pack W8 into bit rows (the B200 counterpart of
 * the compressed W' of L381 / Alg. 2 line 6) and check the structural
 * invariants w_ij = w_ji (L306) and no intra-cluster or padding edges (L145).
 * Asynchronous and stream-ordered: one kernel, no host synchronisation.  Its
 * last CTA publishes the outcome into pinned host memory; gb_seal_status
 * reports it.  Decodes may be issued right away (stream-ordered after the
 * seal); a gb_decode issued after the outcome reached the host refuses a W
 * that broke the invariants (GB_ESTATE).
 */
int gb_seal(gb_net *net, void *stream);

/*
 * gb_seal_status -- wait for the most recent gb_seal and report its outcome:
 * GB_OK; GB_EINVAL if W8 breaks an invariant (the net is then unsealed) or if
 * gb_store calls between the previous seal (or gb_clear) and this one skipped
 * messages with invalid symbols (the net IS sealed; the message says how
 * many); GB_ESTATE if no seal was issued.  Blocks the calling thread only;
 * repeated calls report the same seal's outcome until the next gb_seal.
 */
int gb_seal_status(gb_net *net);

/*
 * gb_decode -- retrieve k probes in one batch (Eq.(11)
 * S^t = W V^t: the columns are independent, so results do not depend on the
 * batch split).
 *   probes      uint16_t[k][c]; GB_ERASED marks an erased cluster.
 *   rule        GB_SUM_OF_SUM: V^0 = known one-hot, erased 0 (L197); rounds
 *                 s = W v + gamma v, keep every per-cluster maximiser (ties
 *                 all kept; a cluster whose max is 0 activates all its real
 *                 neurons, readings R3-R4).
 *               GB_SUM_OF_MAX: V^0 = known one-hot, erased all 1 (L270-271);
 *                 rounds of Eq.(6)-(7), synchronous.
 *               GB_HYBRID: Alg. 2 -- one sum-of-sum pass from V^0 (erased 0)
 *                 keeps erased neurons with exactly C-e signals, then
 *                 sum-of-max rounds on erased clusters only (known clusters
 *                 frozen) until the erased clusters stop changing.
 *   gamma       reinforcement factor (Eq.(3)), 0 <= gamma <= 65535;
 *               must be > 0 for SUM_OF_MAX / HYBRID (Thm 1), where any
 *               positive value gives identical results.
 *   max_iters   maximum number of rounds, 1..65535 (paper runs use 20,
 *               L700; reading R5).
 *   out_state   uint32_t[k][c*Wc]   final V (see "decoded state" above)
 *   out_iters   uint16_t[k]         rounds executed, including the round that
 *                                   showed no change; hybrid counts only its
 *                                   sum-of-max rounds (0 when nothing is
 *                                   erased); reading R6
 *   out_status  uint8_t[k]          GB_CONVERGED / GB_MAX_ITERS / GB_INVALID
 * Synchronous rounds (reading R14).  Returns GB_ESTATE if the net is not
 * sealed, GB_EINVAL for bad rule/gamma/max_iters/k or NULL buffers.
 * k == 0 is a no-op.
 */
int gb_decode(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma,
              int max_iters, uint32_t *out_state, uint16_t *out_iters,
              uint8_t *out_status, void *stream);

/*
 * gb_decode_ex -- gb_decode with option flags (GB_FLAG_*); flags == 0 is
 * gb_decode.  Unknown flag bits -> GB_EINVAL.
 */
int gb_decode_ex(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma,
                 int max_iters, unsigned flags, uint32_t *out_state, uint16_t *out_iters,
                 uint8_t *out_status, void *stream);

/*
 * gb_decode_symbols -- gb_decode_ex, but instead of the state bits it returns the
 * retrieved message: for every probe and cluster the index l of the cluster's only
 * active neuron in the final state, GB_ERASED when no neuron is active and
 * GB_AMBIGUOUS when several are (the network "retrieves" the
 * message when one neuron per cluster remains; reading R16: success is
 * unique exact recovery).  Same decode, rounds and status as gb_decode_ex; only the
 * output representation differs (2 bytes per cluster instead of the cluster's
 * padded bits: 16 vs 128 bytes per probe at c=8 l=128, 32 vs 512 at c=16 l=256),
 * which is what a host-buffer caller copies back over PCIe.
 *   out_symbols uint16_t[k][c]  row-major; GB_INVALID probes get GB_ERASED rows
 *   the other arguments, pointer rules (all device or all host; host buffers are
 *   staged in chunks and the call blocks), errors and concurrency as gb_decode_ex.
 * Implementation: the decode kernels write the state into call-private scratch
 * (n_padded/8 bytes per probe, per staged chunk for host buffers) and one pass
 * maps each cluster block to its symbol.
 */
int gb_decode_symbols(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma,
                      int max_iters, unsigned flags, uint16_t *out_symbols, uint16_t *out_iters,
                      uint8_t *out_status, void *stream);

/* gb_info -- shape and bookkeeping; any out pointer may be NULL.
 * stored_count counts messages passed to gb_store since create/clear.      */
int gb_info(gb_net *net, int *c, int *l, int *n_padded, int64_t *stored_count);

/* gb_launch_count -- number of CUDA kernels this handle has launched so far
 * (diagnostics: bench.py reports the kernels launched in its timed region). */
int gb_launch_count(gb_net *net, int64_t *launches);

/* gb_decode_kernel -- name of the kernel gb_decode launches for `rule` on
 * this handle's shape (diagnostics for profiling and roofline reports). */
const char *gb_decode_kernel(gb_net *net, int rule);

/* gb_last_error -- thread-local message for the last failing call. */
const char *gb_last_error(void);

/* gb_version -- library version string. */
const char *gb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GB_H */
