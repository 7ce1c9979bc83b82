// gb_internal.h -- private declarations shared by libgb's translation units.
// Product code only (the oracle never includes this).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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
    unsigned long long *dcount;  // 16-byte device status: [0, 8) invalid stored messages,
    unsigned *dflag;             // [8, 12) error flags (dflag points into the same allocation),
                                 // [12, 16) edge count of W (both directions, counted by seal)
    void *hstat;                 // 16-byte pinned copy of the status (gb_seal)
    double density;              // edges / (C (C-1) L^2) of the sealed W (kernel heuristics)
    int64_t stored;
    bool sealed;
    // host-staging scratch (gb_decode / gb_store with host pointers)
    void *stage;
    size_t stage_bytes;
    cudaStream_t stage_stream[2];
    cudaEvent_t stage_event[4];
    int64_t launches;     // kernels launched by this handle (diagnostics)
    alignas(64) unsigned char wmap[128];   // CUtensorMap of W8 for the tensor-core SOS kernel
    bool wmap_ok;
    uint8_t *w8g;                          // W8 + gamma*I (B operand of sos_tc2_kernel), lazily built
    alignas(64) unsigned char wmap_g[128];
    alignas(64) unsigned char wmap_g2[128];  // W8g map with the CTA-pair kernel's box (half the rows)
    bool wmap_g2_ok;
    bool wmap_g_ok;                          // wmap_g encoded (sos_tc2 / pair kernels)
    alignas(64) unsigned char wmap_g3[128];  // W8g map with the streamed-A kernel's box
    bool wmap_g3_ok;
    int wmap_g3_br;                          // box rows wmap_g3 was encoded with
    uint8_t *w4;                             // W8 + gamma*I as packed e2m1 (B operand of sos_fp4_kernel)
    alignas(64) unsigned char w4map[128];
    unsigned long long w4_gen;
    int w4_gamma;
    alignas(64) unsigned char omap[128];     // out_state map of decode_hyb8_kernel (cached per buffer, k)
    bool omap_ok;
    const void *omap_ptr;
    int64_t omap_k;
    alignas(64) unsigned char wmap_som[128]; // W8 map for the tensor-core sum-of-max kernel
    bool wmap_som_ok;
    int w8g_gamma;
    unsigned long long seal_gen, w8g_gen;  // W8g is valid for (seal generation, gamma)
    unsigned long long *queue;             // device work counter (slot-refill kernels)
    uint32_t *vscratch;                    // SOS state scratch when it does not fit shared memory
    int64_t *ovf;                          // hybrid probes queued for the wide-slot smem kernel
    int64_t ovf_cap;
    unsigned long long *ovf_count;
    size_t vscratch_bytes;
    uint32_t *xscratch;                    // next-state scratch of the thread-per-probe L2 kernel
    size_t xscratch_bytes;
    uint32_t *spart;                       // per-chunk partial bit matrices of the privatised store
    size_t spart_bytes;
};

namespace gb {

// Launchers (return cudaError_t of the launch).
cudaError_t launch_store(gb_net *net, const uint16_t *msgs, int64_t m, cudaStream_t st);
cudaError_t launch_seal(const gb_net *net, cudaStream_t st);
cudaError_t launch_or_bits(gb_net *net, const uint32_t *bits, int64_t count, cudaStream_t st);
bool decode_smem_supported(const Shape &s, int rule);
bool decode_l2_supported(const Shape &s, int rule);
// thread-per-probe L2 kernel (gb_decode_l2t.cu): probes needing more slots than it
// holds are appended to net->ovf (decode_l2_kernel decodes them in list mode).
bool decode_l2t_supported(const Shape &s, int rule);
cudaError_t launch_decode_l2t(gb_net *net, const uint16_t *probes, int64_t k, int rule, int max_iters,
                              uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st);
cudaError_t launch_decode_l2(gb_net *net, const uint16_t *probes, int64_t k, int rule, int max_iters,
                             uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st);
bool sos_tc_supported(const Shape &s);
bool sos_tc2_supported(const Shape &s);
bool sos_tc_make_map(gb_net *net);
bool sos_encode_map(gb_net *net, void *gaddr, int box_rows, unsigned char *out);
// CTA-pair (cta_group::2) sum-of-sum kernel, gb_decode_sos_2cta.cu; the caller
// has built W8g = W8 + gamma*I (gamma_epi = gamma when gamma > 255, else 0).
bool sos_2cta_enabled(const Shape &s);
int sos_2cta_box_rows(const Shape &s);
cudaError_t launch_sos_2cta(gb_net *net, int gamma_epi, int cyc, const uint16_t *probes, int64_t k, int max_iters,
                            uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st);
// C = 8, Wc = 4 hybrid decode of the probes with e <= 4 (gb_decode_hyb8.cu); the
// others are appended to net->ovf.
bool decode_hyb8_supported(const Shape &s, int rule, int64_t k, const void *state);
cudaError_t launch_decode_hyb8(gb_net *net, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                               uint16_t *iters, uint8_t *status, cudaStream_t st);
// Streamed-A sum-of-sum kernel for 1024 < n_p <= 4096 (gb_decode_sos_tc3.cu); the
// caller has built W8g = W8 + gamma*I and its tensor map (box rows from plan3).
bool plan3(const Shape &s, int gamma, void *params, size_t &smem);
int plan3_box_rows(const void *params);
bool sos_tc3_enabled(const Shape &s);
bool sos_tc3_pair(const Shape &s);   // the streamed-A kernel runs on CTA pairs
cudaError_t launch_sos_tc3(gb_net *net, int gamma, int cyc, const void *map, const uint16_t *probes, int64_t k,
                           int max_iters, uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st);
// cyc = 1: period-2 cycle exit (GB_FLAG_CYCLE_EXIT) in every sum-of-sum kernel
// sum-of-sum on block-scaled FP4 tensor cores (gb_decode_sos_fp4.cu)
bool sos_fp4_enabled(const Shape &s, int gamma);
cudaError_t launch_sos_fp4(gb_net *net, int gamma, int cyc, const uint16_t *probes, int64_t k, int max_iters,
                           uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st);
// exact sum-of-max on the tensor cores (gb_decode_som_tc.cu, N2), opt-in with GB_SOM_TC=1
bool som_tc_enabled(const Shape &s);
cudaError_t launch_som_tc(gb_net *net, const uint16_t *probes, int64_t k, int max_iters, uint32_t *state,
                          uint16_t *iters, uint8_t *status, cudaStream_t st);
cudaError_t launch_decode_sos_tc(gb_net *net, const uint16_t *probes, int64_t k, int gamma, int max_iters,
                                 int cyc, uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st);
cudaError_t launch_decode(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma,
                          int max_iters, int cyc, uint32_t *state, uint16_t *iters, uint8_t *status,
                          cudaStream_t st);

}  // namespace gb
