// gb_internal.h -- private declarations shared by libgb's translation units.
// Product code only (the oracle never includes this).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

#include "../../include/gb.h"

namespace gb {

constexpr int kMaxClusters = 64;
constexpr int kMaxPadded = 8192;      // n_padded limit (W8 = 64 MiB)
constexpr uint16_t kErased = 0xFFFFu;

// Device-side error bits (gb_net::dflag).
enum : unsigned {
    kFlagStoreInvalid = 1u,   // counted separately in dcount[0]
    kFlagAsym = 2u,           // W8 not symmetric
    kFlagIntra = 4u,          // edge inside a cluster / on the diagonal
    kFlagPad = 8u,            // edge touching a padding neuron
    kFlagNotBinary = 16u      // W8 byte not in {0,1}
};

// Seal status as the last CTA of a seal kernel publishes it (mapped pinned host memory).
struct Status {
    unsigned long long gen;        // seal generation this status belongs to
    unsigned long long invalid;    // invalid stored messages since create/clear
    unsigned flags;                // structural error flags (kFlagAsym | kFlagIntra | ...)
    unsigned edges;                // set entries of W (both directions)
};

// Kernel-selection options of a handle (gb_set_option; GB_OPT_* in gb.h).
constexpr int kNumOptions = 9;

// One W8 + gamma*I operand (gamma folded into the int8 diagonal, 0..255).
constexpr int kGammaVariants = 4;
struct GammaVariant {
    int gfold = -1;
    unsigned long long gen = ~0ull;   // seal generation it was built from
    uint8_t *w8g = nullptr;
    cudaEvent_t ready = nullptr;      // recorded after its build kernel
    int nmaps = 0;
    int map_rows[4] = {0, 0, 0, 0};
    alignas(64) unsigned char maps[4][128];   // CUtensorMaps of w8g, by box rows
    unsigned long long last_use = 0;
};

struct Shape {
    int C;      // clusters
    int L;      // neurons per cluster
    int Wc;     // 32-bit words per cluster = ceil(L/32)
    int Lp;     // padded cluster size = 32*Wc
    int np;     // padded neuron count = C*Lp
    int nw;     // words per state / per bit row = C*Wc
};

}  // namespace gb

struct gb_net {
    gb::Shape s;
    int device;
    int sm_count;
    uint8_t *w8;          // [np][np] u8, row-major
    uint32_t *wb;         // [np][nw] bit rows
    uint32_t *wu;         // 2 x [C][C][Wc] cluster unions: block t of the OR of all rows of cluster
                          // s (the push cover of a full source cluster), built by the seal into
                          // buffer (generation & 1) -- wu_of(net, net->seal_gen) is the current one
    // Device status words (one 32-byte allocation):
    //   [0, 8) invalid stored messages since create/clear (store kernels; reset by gb_clear)
    //   [8, 12) structural error flags of the running seal, [12, 16) its edge count,
    //   [16, 20) CTAs of the running seal that have finished (the last one publishes + resets)
    unsigned long long *dcount;
    unsigned *dflag;             // = dcount + 8 bytes
    gb::Status *hstat;           // mapped pinned host memory: the seal kernel publishes here
    gb::Status *hstat_dev;       // its device alias
    cudaEvent_t seal_event;      // recorded after each seal kernel
    std::mutex smu;              // seal-status resolution (host side)
    unsigned long long seal_gen = 0;         // seals enqueued (generation of the sealed W)
    unsigned long long seal_resolved = 0;    // last seal whose status the host has read
    unsigned long long invalid_reported = 0; // invalid-message count already reported
    unsigned long long clear_epoch = 0;      // gb_clear calls (they reset the device count)
    unsigned long long seal_epoch = 0;       // clear_epoch when the latest seal was issued
    unsigned long long reported_epoch = 0;   // epoch invalid_reported belongs to
    int seal_rc = 0;                         // outcome of the latest resolved seal
    char seal_msg[200] = "";
    std::atomic<double> density{0.0};        // edges / (C (C-1) L^2) of the last resolved seal (heuristics)
    int64_t stored = 0;
    std::atomic<bool> sealed{false};         // a seal is enqueued and no W change followed
    std::atomic<bool> seal_broken{false};    // the last resolved seal found broken invariants
    // kernel-selection options (gb_set_option), read by decodes
    std::atomic<int> opt[gb::kNumOptions];
    // stream-ordered per-call scratch (work counters, overflow lists, state scratch, staging)
    cudaMemPool_t pool = nullptr;
    // host-buffer staging (gb_decode / gb_store with host pointers): serialised per handle
    std::mutex stage_mu;
    // host-buffer decode pipeline: [0] copy-in, [1] compute, [2] copy-out streams; per staging
    // slot the events "copied in", "decoded", "copied out"
    static constexpr int kStageSlots = 3;
    cudaStream_t stage_stream[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t stage_event = nullptr;
    cudaEvent_t slot_ev[kStageSlots][3] = {};
    std::atomic<long long> launches{0};      // kernels launched by this handle (diagnostics)
    alignas(64) unsigned char wmap[128];     // CUtensorMap of W8 for the 4-warp SOS kernel
    bool wmap_ok = false;
    alignas(64) unsigned char wmap_som[128]; // W8 map for the tensor-core sum-of-max kernel
    bool wmap_som_ok = false;
    std::mutex som_mu;
    // W8 + gamma*I variants (B operand of the warp-specialised SOS kernels), one per folded gamma
    std::mutex gmu;
    gb::GammaVariant gvar[gb::kGammaVariants];
    unsigned long long guse = 0;
};

namespace gb {

inline uint32_t *wu_of(const gb_net *net, unsigned long long gen) {
    return net->wu + (size_t)(gen & 1ull) * net->s.C * net->s.C * net->s.Wc;
}

// One store / decode call: the caller's stream and the call's private device scratch,
// allocated stream-ordered from the handle's memory pool and released (stream-ordered)
// when the call object goes out of scope.  Nothing a kernel writes lives in the handle,
// so concurrent decodes on one handle (distinct streams, host threads) cannot race
// (SURVEY.md §8.b "Concurrency").
struct Call {
    gb_net *net;
    cudaStream_t st;
    cudaError_t err = cudaSuccess;
    Call(gb_net *n, cudaStream_t s) : net(n), st(s) {}
    Call(const Call &) = delete;
    Call &operator=(const Call &) = delete;
    ~Call();
    void *alloc(size_t bytes);     // nullptr on failure (err set)
    template <class T> T *alloc_n(size_t n) { return static_cast<T *>(alloc(n * sizeof(T))); }
    // [0] work queue of the slot-refill kernels, [1] overflow count, [2] work queue of a list-mode
    // kernel decoding the overflow; zeroed once per call
    unsigned long long *counters();
    // overflow list of probe indices (k entries) for the two-pass bit kernels
    int64_t *ovf(int64_t k);
    int opt(int o) const { return net->opt[o].load(std::memory_order_relaxed); }
    void launched(int n = 1) { net->launches.fetch_add(n, std::memory_order_relaxed); }

  private:
    void *blk_[8];
    int nblk_ = 0;
    unsigned long long *counters_ = nullptr;
    int64_t *ovf_ = nullptr;
};

// Option indices (gb.h GB_OPT_*) and defaults.
enum : int {
    kOptSosPair = 0,       // CTA-pair (cta_group::2) sum-of-sum kernels
    kOptSosStreamed = 1,   // streamed-A sum-of-sum kernel for 1024 < n_p <= 4096
    kOptSomTensor = 2,     // exact sum-of-max on the tensor cores (N2)
    kOptHyb8 = 3,          // C = 8 hybrid kernel
    kOptL2t = 4,           // thread-per-probe L2 bit kernel
    kOptHyb8Split = 5,     // C = 8 hybrid kernel: -1 by density, 0 sparse loop, 1 dense rotated layout
    kOptStoreScatter = 6,  // store with scattered byte writes only (no privatised tiles)
    kOptHyb8Rows = 7,      // rows of the dense C = 8 hybrid kernel's first push step: 0 by density, 6..8
    kOptSosBits = 8,       // sum-of-sum on the CUDA cores for sparse states: -1 by density, 0 off, 1 on
};
int option_default(int o);

// Launchers (return cudaError_t of the launch; cudaErrorNotSupported = shape not taken).
cudaError_t launch_store(Call &cl, const uint16_t *msgs, int64_t m);
cudaError_t launch_seal(gb_net *net, cudaStream_t st);
cudaError_t launch_or_bits(Call &cl, const uint32_t *bits, int64_t count);
cudaError_t launch_or_multimem(Call &cl, const uint32_t *mc);
int64_t upper_words(const Shape &s);   // words of one packed upper-triangle set
cudaError_t launch_pack_upper(Call &cl, uint32_t *out);
cudaError_t launch_or_upper(Call &cl, const uint32_t *sets, int64_t count);
bool decode_smem_supported(const Shape &s, int rule);
bool decode_l2_supported(const Shape &s, int rule);
// thread-per-probe L2 kernel (gb_decode_l2t.cu): probes needing more slots than it
// holds are appended to the call's overflow list (decode_l2_kernel decodes them in list mode).
bool decode_l2t_supported(const gb_net *net, int rule);
cudaError_t launch_decode_l2t(Call &cl, const uint16_t *probes, int64_t k, int rule, int max_iters,
                              uint32_t *state, uint16_t *iters, uint8_t *status);
cudaError_t launch_decode_l2(Call &cl, const uint16_t *probes, int64_t k, int rule, int max_iters,
                             uint32_t *state, uint16_t *iters, uint8_t *status);
cudaError_t launch_decode_smem(Call &cl, const uint16_t *probes, int64_t k, int rule, int max_iters,
                               uint32_t *state, uint16_t *iters, uint8_t *status);
cudaError_t launch_decode_generic(Call &cl, const uint16_t *probes, int64_t k, int rule, int gamma,
                                  int max_iters, int cyc, uint32_t *state, uint16_t *iters, uint8_t *status);
cudaError_t launch_decode_generic_list(Call &cl, const uint16_t *probes, int64_t k, const int64_t *list,
                                       const unsigned long long *count, int rule, int gamma, int max_iters,
                                       uint32_t *state, uint16_t *iters, uint8_t *status);
// Sum-of-sum on the CUDA cores for sparse states (gb_decode_sos_bits.cu): C <= 8, n_p <= 1024.
bool sos_bits_supported(const Shape &s, int gamma, int cyc);
bool sos_bits_chosen(const gb_net *net, int gamma, int cyc);   // option / density (gb_api.cu)
cudaError_t launch_sos_bits(Call &cl, const uint16_t *probes, int64_t k, int gamma, int max_iters,
                            uint32_t *state, uint16_t *iters, uint8_t *status);
bool sos_tc_supported(const Shape &s);
bool sos_tc2_supported(const Shape &s);
bool sos_tc_make_map(gb_net *net);
bool sos_encode_map(const gb_net *net, void *gaddr, int box_rows, unsigned char *out);
// The W8 + gamma*I operand for gamma (folded when <= 255), built (once per seal and
// gamma) on / ordered before the call's stream, and its tensor map with `box_rows` rows.
cudaError_t gamma_operand(Call &cl, int gamma, int box_rows, const void **map);
// CTA-pair (cta_group::2) sum-of-sum kernel, gb_decode_sos_2cta.cu; `map` is the W8 + gamma*I
// operand (gamma_epi = gamma when gamma > 255, else 0).
bool sos_2cta_enabled(const gb_net *net);
int sos_2cta_box_rows(const Shape &s);
cudaError_t launch_sos_2cta(Call &cl, const void *map, int gamma_epi, int cyc, const uint16_t *probes, int64_t k,
                            int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status,
                            const int64_t *list = nullptr, const unsigned long long *list_count = nullptr);
// The CTA-pair SOS kernel in list mode (the *count probes queued in list; k bounds the count);
// cudaErrorNotSupported when the pair kernel does not take the shape.
cudaError_t launch_sos_pair_list(Call &cl, const uint16_t *probes, int64_t k, const int64_t *list,
                                 const unsigned long long *count, int gamma, int max_iters, uint32_t *state,
                                 uint16_t *iters, uint8_t *status);
// C = 8, Wc = 4 hybrid decode of the probes with e <= 4 (gb_decode_hyb8.cu); the
// others are appended to the overflow list `ovf`.
bool decode_hyb8_supported(const gb_net *net, int rule, int64_t k, const void *state);
bool decode_hyb8_rotated(const gb_net *net);   // dense W: decode_hyb8r_kernel
cudaError_t launch_decode_hyb8(Call &cl, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                               uint16_t *iters, uint8_t *status, int64_t *ovf, unsigned long long *ovf_count);
// Streamed-A sum-of-sum kernel for 1024 < n_p <= 4096 (gb_decode_sos_tc3.cu); `map` is the
// W8 + gamma*I operand with plan3's box rows.
bool plan3(const gb_net *net, int gamma, void *params, size_t &smem);
int plan3_box_rows(const void *params);
bool sos_tc3_enabled(const gb_net *net);
bool sos_tc3_pair(const gb_net *net);   // the streamed-A kernel runs on CTA pairs
cudaError_t launch_sos_tc3(Call &cl, int gamma, int cyc, const void *map, const uint16_t *probes, int64_t k,
                           int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status);
// cyc = 1: period-2 cycle exit (GB_FLAG_CYCLE_EXIT) in every sum-of-sum kernel
// exact sum-of-max on the tensor cores (gb_decode_som_tc.cu, N2), option GB_OPT_SOM_TENSOR
bool som_tc_enabled(const gb_net *net);
cudaError_t launch_som_tc(Call &cl, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                          uint16_t *iters, uint8_t *status);
cudaError_t launch_decode_sos_tc(Call &cl, const uint16_t *probes, int64_t k, int gamma, int max_iters,
                                 int cyc, uint32_t *state, uint16_t *iters, uint8_t *status);
cudaError_t launch_decode(Call &cl, const uint16_t *probes, int64_t k, int rule, int gamma,
                          int max_iters, int cyc, uint32_t *state, uint16_t *iters, uint8_t *status);
// gb_decode_symbols' output pass (gb_symbols.cu): state bits -> one uint16 per cluster
cudaError_t launch_symbols(Call &cl, const uint32_t *state, int64_t k, uint16_t *out);

}  // namespace gb
