/*
 * gb_oracle.c -- plain CPU oracle for Gripon-Berrou (GBNN) store and decode.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1303_7032_b200/csrc, include/gb.h) and never includes them.
 *
 * Everything is a literal transcription of PAPER.md (arXiv:1303.7032) on
 * 0/1 byte arrays: no bit packing, no early exits, no reordering.  The
 * output is then *formatted* (packed into the cluster-padded bit layout the
 * C-ABI returns) so results compare byte for byte.
 *
 * Notation: C clusters of L neurons, n = C*L,
 * neuron(c,l) <-> i = c*L + l (0-based, reading R1).
 * W is n x n u8, W[i*n+j] = w_ij in {0,1}; the diagonal is NOT stored,
 * gamma is added at decode (reading R2, algebraically identical to the
 * gamma diagonal of PAPER.md L330-336).
 *
 * Iteration semantics (readings R5-R7, R14): synchronous rounds; max_iters
 * T bounds the number of rounds (score+select passes); a probe's iteration
 * count is the number of rounds executed including the round that shows no
 * change; status CONVERGED when V^r == V^{r-1} for some r <= T, else
 * MAX_ITERS with V^T returned.  Hybrid counts only its bail-out rounds.
 * Optional (flag OR_CYCLE_EXIT, SOS only, SPEC S:L304 design
 * decision): a round r >= 2 whose state repeats the state of round r-2
 * (V^r == V^{r-2} != V^{r-1}, the period-2 oscillation PAPER.md L515-517
 * exhibits) stops the probe with status CYCLE and V^r returned.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_ERASED 0xFFFFu
enum { OR_SOS = 0, OR_SOM = 1, OR_HYBRID = 2 };
enum { OR_CONVERGED = 0, OR_MAX_ITERS = 1, OR_INVALID = 2, OR_CYCLE = 3 };
enum { OR_CYCLE_EXIT = 1 };

/* ------------------------------------------------------------------ */
/* STORE  ("we add edges to the network connecting all
 * pairs of nodes which are activated"; Eq.(1)).
 * For every message and every ordered cluster pair c != c':
 *     W[(c,m_c)][(c',m_c')] := 1.
 * A message with a symbol >= L is skipped (no edge stored) and counted.
 * Returns the number of skipped (invalid) messages.                    */
int64_t oracle_store(uint8_t *W, int C, int L, const uint16_t *msgs, int64_t M)
{
    const int64_t n = (int64_t)C * L;
    int64_t invalid = 0;
    for (int64_t m = 0; m < M; ++m) {
        const uint16_t *msg = msgs + m * C;
        int ok = 1;
        for (int c = 0; c < C; ++c)
            if (msg[c] >= L) ok = 0;
        if (!ok) { ++invalid; continue; }
        for (int c = 0; c < C; ++c)
            for (int c2 = 0; c2 < C; ++c2)
                if (c2 != c) {
                    int64_t i = (int64_t)c * L + msg[c];
                    int64_t j = (int64_t)c2 * L + msg[c2];
                    W[i * n + j] = 1;
                }
    }
    return invalid;
}

/* ------------------------------------------------------------------ */
/* Output formatting: cluster-padded bits, Wc = ceil(L/32) words per
 * cluster, bit l%32 of word c*Wc + l/32; padding bits are 0.           */
static void pack_state(const uint8_t *V, int C, int L, uint32_t *out)
{
    const int Wc = (L + 31) / 32;
    memset(out, 0, sizeof(uint32_t) * (size_t)C * Wc);
    for (int c = 0; c < C; ++c)
        for (int l = 0; l < L; ++l)
            if (V[(int64_t)c * L + l])
                out[c * Wc + l / 32] |= 1u << (l % 32);
}

static int same(const uint8_t *a, const uint8_t *b, int64_t n)
{
    for (int64_t i = 0; i < n; ++i)
        if (a[i] != b[i]) return 0;
    return 1;
}

/* SOS round, Eq.(3)-(5):
 *   s_i = gamma*v_i + sum_j w_ji v_j          (literal sum over all j)
 *   s_c,max = max_l s_(c,l);  v'_(c,l) = [s_(c,l) == s_c,max]
 * (all maximizers kept, reading R3; a cluster whose max is 0 activates
 * all its neurons, reading R4).                                          */
static void sos_round(const uint8_t *W, int C, int L, int gamma,
                      const uint8_t *V, uint8_t *Vn, int64_t *S)
{
    const int64_t n = (int64_t)C * L;
    for (int64_t i = 0; i < n; ++i) {
        int64_t s = (int64_t)gamma * V[i];
        for (int64_t j = 0; j < n; ++j)
            s += (int64_t)W[j * n + i] * V[j];
        S[i] = s;
    }
    for (int c = 0; c < C; ++c) {
        int64_t mx = S[(int64_t)c * L];
        for (int l = 1; l < L; ++l)
            if (S[(int64_t)c * L + l] > mx) mx = S[(int64_t)c * L + l];
        for (int l = 0; l < L; ++l)
            Vn[(int64_t)c * L + l] = (S[(int64_t)c * L + l] == mx);
    }
}

/* SOM score + select for neuron i, Eq.(6)-(7):
 *   s_i = gamma*v_i + sum_{c'=1..C} max_{l'} (v_(c',l') w_(c'l')(i))
 *   v'_i = [s_i == gamma + C - 1]
 * The c' = c(i) term is max over intra-cluster w, which is 0 by Eq.(1)
 * (no intra-cluster edges, diagonal not stored).  Literal over all c'.   */
static uint8_t som_neuron(const uint8_t *W, int C, int L, int gamma,
                          const uint8_t *V, int64_t i)
{
    const int64_t n = (int64_t)C * L;
    int64_t s = (int64_t)gamma * V[i];
    for (int c2 = 0; c2 < C; ++c2) {
        int64_t mx = 0;
        for (int l2 = 0; l2 < L; ++l2) {
            int64_t j = (int64_t)c2 * L + l2;
            int64_t a = (int64_t)V[j] * W[j * n + i];
            if (a > mx) mx = a;
        }
        s += mx;
    }
    return (uint8_t)(s == (int64_t)gamma + C - 1);
}

/* Work counter (oracle-only, for DESIGN.md's W-row bytes): the
 * bail-out-early walk of PAPER.md L445-451 for active neuron i over the
 * clusters in `scope` other than c(i), ascending; counts L-bit blocks read
 * until (and including) the first silent cluster.                        */
static int64_t bailout_blocks(const uint8_t *W, int C, int L, const uint8_t *V,
                              int64_t i, const uint8_t *scope)
{
    const int64_t n = (int64_t)C * L;
    const int ci = (int)(i / L);
    int64_t blocks = 0;
    for (int c2 = 0; c2 < C; ++c2) {
        if (c2 == ci || !scope[c2]) continue;
        ++blocks;
        int hit = 0;
        for (int l2 = 0; l2 < L; ++l2) {
            int64_t j = (int64_t)c2 * L + l2;
            if (V[j] && W[j * n + i]) hit = 1;
        }
        if (!hit) break;
    }
    return blocks;
}

typedef struct {
    uint8_t *V, *Vn, *V2;
    int64_t *S;
    uint8_t *scope;
} scratch_t;

/* Decode one probe.  Returns status; writes rounds to *iters. */
static int decode_one(const uint8_t *W, int C, int L, const uint16_t *p,
                      int rule, int gamma, int T, int flags, scratch_t *sc,
                      uint16_t *iters, int64_t *blocks)
{
    const int64_t n = (int64_t)C * L;
    uint8_t *V = sc->V, *Vn = sc->Vn;
    int64_t work = 0;
    int e = 0;
    for (int c = 0; c < C; ++c) {
        if (p[c] == OR_ERASED) { ++e; continue; }
        if (p[c] >= L) {                      /* invalid symbol */
            memset(V, 0, (size_t)n);
            *iters = 0;
            if (blocks) *blocks = 0;
            return OR_INVALID;
        }
    }
    for (int c = 0; c < C; ++c) sc->scope[c] = (p[c] == OR_ERASED);

    if (rule == OR_SOS) {
        /* V^0: known clusters one-hot, erased clusters 0. */
        for (int c = 0; c < C; ++c)
            for (int l = 0; l < L; ++l)
                V[(int64_t)c * L + l] = (p[c] != OR_ERASED && p[c] == l);
        /* Alg. 1, max_iters = max rounds (R5). */
        for (int r = 1; r <= T; ++r) {
            sos_round(W, C, L, gamma, V, Vn, sc->S);
            int conv = same(V, Vn, n);
            /* V2 holds V^{r-2} (valid for r >= 2) */
            int cyc = (flags & OR_CYCLE_EXIT) && r >= 2 && same(Vn, sc->V2, n);
            memcpy(sc->V2, V, (size_t)n);
            memcpy(V, Vn, (size_t)n);
            work += 1;
            if (conv) { *iters = (uint16_t)r; if (blocks) *blocks = work; return OR_CONVERGED; }
            if (cyc) { *iters = (uint16_t)r; if (blocks) *blocks = work; return OR_CYCLE; }
        }
        *iters = (uint16_t)T;
        if (blocks) *blocks = work;
        return OR_MAX_ITERS;
    }

    if (rule == OR_SOM) {
        /* V^0: erased clusters all 1, known one-hot. */
        for (int c = 0; c < C; ++c)
            for (int l = 0; l < L; ++l)
                V[(int64_t)c * L + l] = (p[c] == OR_ERASED) ? 1 : (p[c] == l);
        uint8_t *all = (uint8_t *)malloc((size_t)C);
        for (int c = 0; c < C; ++c) all[c] = 1;
        for (int r = 1; r <= T; ++r) {
            for (int64_t i = 0; i < n; ++i) {
                Vn[i] = som_neuron(W, C, L, gamma, V, i);
                if (V[i]) work += bailout_blocks(W, C, L, V, i, all);
            }
            int conv = same(V, Vn, n);
            memcpy(V, Vn, (size_t)n);
            if (conv) { free(all); *iters = (uint16_t)r; if (blocks) *blocks = work; return OR_CONVERGED; }
        }
        free(all);
        *iters = (uint16_t)T;
        if (blocks) *blocks = work;
        return OR_MAX_ITERS;
    }

    /* HYBRID, Alg. 2. */
    /* L620: all neurons inactive in erased clusters; known one-hot.      */
    for (int c = 0; c < C; ++c)
        for (int l = 0; l < L; ++l)
            V[(int64_t)c * L + l] = (p[c] != OR_ERASED && p[c] == l);
    if (e == 0) {                     /* nothing erased: 0 rounds (R6). */
        *iters = 0;
        if (blocks) *blocks = 0;
        return OR_CONVERGED;
    }
    /* L621: S^0 = W V^0 (sum-of-sum score, gamma*v term included).      */
    for (int64_t i = 0; i < n; ++i) {
        int64_t s = (int64_t)gamma * V[i];
        for (int64_t j = 0; j < n; ++j)
            s += (int64_t)W[j * n + i] * V[j];
        sc->S[i] = s;
    }
    /* L622-624: in erased clusters keep neurons with exactly C-e signals. */
    for (int c = 0; c < C; ++c)
        if (p[c] == OR_ERASED)
            for (int l = 0; l < L; ++l)
                V[(int64_t)c * L + l] = (sc->S[(int64_t)c * L + l] == (int64_t)(C - e));
    work += (int64_t)(C - e) * e;    /* prune reads (C-e)*e blocks */
    /* L626-632: bail-out-early (= SOM, Thm 1) on erased-cluster neurons;
     * non-erased clusters are kept as they are (frozen); stop when the
     * erased clusters no longer change.                                  */
    for (int r = 1; r <= T; ++r) {
        memcpy(Vn, V, (size_t)n);
        for (int c = 0; c < C; ++c) {
            if (p[c] != OR_ERASED) continue;
            for (int l = 0; l < L; ++l) {
                int64_t i = (int64_t)c * L + l;
                Vn[i] = som_neuron(W, C, L, gamma, V, i);
                if (V[i]) work += bailout_blocks(W, C, L, V, i, sc->scope);
            }
        }
        int conv = same(V, Vn, n);
        memcpy(V, Vn, (size_t)n);
        if (conv) { *iters = (uint16_t)r; if (blocks) *blocks = work; return OR_CONVERGED; }
    }
    *iters = (uint16_t)T;
    if (blocks) *blocks = work;
    return OR_MAX_ITERS;
}

/* Batch decode.  probes uint16 [K][C]; out_state uint32 [K][C*Wc];
 * out_iters uint16 [K]; out_status uint8 [K]; out_blocks int64 [K] or NULL.
 * Returns 0, or -1 on bad arguments (rule, gamma, T).  OpenMP over probes
 * (independent columns of Eq.(11)).                   */
int oracle_decode_flags(const uint8_t *W, int C, int L, const uint16_t *probes,
                        int64_t K, int rule, int gamma, int T, int flags,
                        uint32_t *out_state, uint16_t *out_iters,
                        uint8_t *out_status, int64_t *out_blocks);

int oracle_decode(const uint8_t *W, int C, int L, const uint16_t *probes,
                  int64_t K, int rule, int gamma, int T,
                  uint32_t *out_state, uint16_t *out_iters,
                  uint8_t *out_status, int64_t *out_blocks)
{
    return oracle_decode_flags(W, C, L, probes, K, rule, gamma, T, 0, out_state,
                               out_iters, out_status, out_blocks);
}

int oracle_decode_flags(const uint8_t *W, int C, int L, const uint16_t *probes,
                        int64_t K, int rule, int gamma, int T, int flags,
                        uint32_t *out_state, uint16_t *out_iters,
                        uint8_t *out_status, int64_t *out_blocks)
{
    if (C < 2 || L < 1 || T < 1 || T > 65535 || gamma < 0) return -1;
    if (rule != OR_SOS && rule != OR_SOM && rule != OR_HYBRID) return -1;
    if (rule != OR_SOS && gamma == 0) return -1;
    const int64_t n = (int64_t)C * L;
    const int nw = C * ((L + 31) / 32);
#pragma omp parallel
    {
        scratch_t sc;
        sc.V = (uint8_t *)malloc((size_t)n);
        sc.Vn = (uint8_t *)malloc((size_t)n);
        sc.V2 = (uint8_t *)malloc((size_t)n);
        sc.S = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
        sc.scope = (uint8_t *)malloc((size_t)C);
#pragma omp for schedule(dynamic, 16)
        for (int64_t k = 0; k < K; ++k) {
            uint16_t it = 0;
            int64_t blk = 0;
            int st = decode_one(W, C, L, probes + k * C, rule, gamma, T, flags, &sc,
                                &it, out_blocks ? &blk : NULL);
            pack_state(sc.V, C, L, out_state + k * nw);
            out_iters[k] = it;
            out_status[k] = (uint8_t)st;
            if (out_blocks) out_blocks[k] = blk;
        }
        free(sc.V); free(sc.Vn); free(sc.V2); free(sc.S); free(sc.scope);
    }
    return 0;
}

/* SOS trajectory for the PAPER.md L515-522 worked example: records
 * s^0..s^{T-1} (int64 [T][n]) and v^0..v^T (u8 [T+1][n]).  Runs exactly
 * T rounds (no convergence stop).                                       */
int oracle_sos_trace(const uint8_t *W, int C, int L, const uint8_t *v0,
                     int gamma, int T, int64_t *S_out, uint8_t *V_out)
{
    const int64_t n = (int64_t)C * L;
    memcpy(V_out, v0, (size_t)n);
    for (int r = 0; r < T; ++r)
        sos_round(W, C, L, gamma, V_out + r * n, V_out + (r + 1) * n, S_out + r * n);
    return 0;
}

/* One literal SOM step (Eq.(6)-(7)) on an arbitrary 0/1 state.          */
int oracle_som_step(const uint8_t *W, int C, int L, const uint8_t *V,
                    int gamma, uint8_t *Vn)
{
    const int64_t n = (int64_t)C * L;
    for (int64_t i = 0; i < n; ++i) Vn[i] = som_neuron(W, C, L, gamma, V, i);
    return 0;
}
