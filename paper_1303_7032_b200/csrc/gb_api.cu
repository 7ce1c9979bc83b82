// gb_api.cu -- the C-ABI of libgb (include/gb.h): handle lifecycle,
// argument validation, error reporting, host-buffer staging and dispatch to
// the sm_100a kernels.  No compute happens on the host: every step of
// store/seal/decode runs in the kernels of gb_store.cu / gb_decode_*.cu.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <new>

#include "gb_internal.h"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(GB_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define GB_CUDA(call, what)                                  \
    do {                                                     \
        cudaError_t _e = (call);                             \
        if (_e != cudaSuccess) return cuda_fail(_e, what);   \
    } while (0)

// Switch to the handle's device for the duration of a call; restore after.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = (cudaSetDevice(dev) == cudaSuccess);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// 1 = device (or managed) memory of `dev`, 0 = host memory, -1 = other device.
int where(const void *p, int dev) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged)
        return a.device == dev ? 1 : -1;
    return 0;
}

// Resolve the outcome of the most recent gb_seal (its status is published by the seal
// kernel into mapped pinned memory).  block = false: only if the seal has completed.
// Returns GB_OK, GB_EINVAL (broken invariants or skipped messages; message set) or
// 1 = still running (block = false).
int resolve_seal(gb_net *net, bool block) {
    std::lock_guard<std::mutex> lk(net->smu);
    if (net->seal_gen == 0) return fail(GB_ESTATE, "gb_seal_status: no seal issued");
    if (net->seal_resolved != net->seal_gen) {
        if (block) {
            cudaError_t e = cudaEventSynchronize(net->seal_event);
            if (e != cudaSuccess) return cuda_fail(e, "gb_seal_status: sync");
        } else {
            const cudaError_t q = cudaEventQuery(net->seal_event);
            if (q == cudaErrorNotReady) return 1;
            if (q != cudaSuccess) return cuda_fail(q, "gb_seal_status: query");
        }
        const volatile gb::Status *h = net->hstat;
        if (h->gen != net->seal_gen) return fail(GB_ECUDA, "gb_seal_status: status of seal %llu not published",
                                                 (unsigned long long)net->seal_gen);
        const unsigned flag = h->flags;
        const unsigned long long inv = h->invalid;
        const double pairs = (double)net->s.C * (net->s.C - 1) * (double)net->s.L * net->s.L;
        net->density.store(pairs > 0 ? h->edges / pairs : 0.0);
        if (net->seal_epoch != net->reported_epoch) {   // gb_clear reset the device count
            net->reported_epoch = net->seal_epoch;
            net->invalid_reported = 0;
        }
        const unsigned long long fresh = inv - net->invalid_reported;
        net->invalid_reported = inv;
        net->seal_resolved = net->seal_gen;
        const unsigned structural = flag & ~gb::kFlagStoreInvalid;
        net->seal_broken = structural != 0;
        net->seal_rc = GB_OK;
        net->seal_msg[0] = 0;
        if (structural) {
            net->sealed = false;
            net->seal_rc = GB_EINVAL;
            snprintf(net->seal_msg, sizeof net->seal_msg, "gb_seal: W8 breaks Eq.(1) invariants:%s%s%s%s",
                     (structural & gb::kFlagNotBinary) ? " non-binary entry" : "",
                     (structural & gb::kFlagAsym) ? " asymmetric" : "",
                     (structural & gb::kFlagIntra) ? " intra-cluster edge" : "",
                     (structural & gb::kFlagPad) ? " padding edge" : "");
        } else if (fresh) {
            net->seal_rc = GB_EINVAL;
            snprintf(net->seal_msg, sizeof net->seal_msg,
                     "gb_seal: %llu stored message(s) had a symbol >= L and were skipped", fresh);
        }
    }
    if (net->seal_rc != GB_OK) return fail(net->seal_rc, "%s", net->seal_msg);
    return GB_OK;
}

}  // namespace

extern "C" {

const char *gb_last_error(void) { return g_err; }

const char *gb_version(void) { return "libgb 0.2 (sm_100a)"; }

int gb_create(int c, int l, int device, gb_net **out) {
    if (!out) return fail(GB_EINVAL, "gb_create: out is NULL");
    *out = nullptr;
    if (c < 2 || l < 1) return fail(GB_EINVAL, "gb_create: need c >= 2 and l >= 1 (got %d, %d)", c, l);
    gb::Shape s;
    s.C = c;
    s.L = l;
    s.Wc = (l + 31) / 32;
    s.Lp = 32 * s.Wc;
    if (c > gb::kMaxClusters || (int64_t)c * s.Lp > gb::kMaxPadded)
        return fail(GB_EUNSUPPORTED, "gb_create: c=%d l=%d exceeds c<=%d, n_padded<=%d", c, l,
                    gb::kMaxClusters, gb::kMaxPadded);
    s.np = c * s.Lp;
    s.nw = c * s.Wc;
    int ndev = 0;
    GB_CUDA(cudaGetDeviceCount(&ndev), "gb_create: cudaGetDeviceCount");
    if (device < 0 || device >= ndev) return fail(GB_EINVAL, "gb_create: device %d of %d", device, ndev);
    cudaDeviceProp prop;
    GB_CUDA(cudaGetDeviceProperties(&prop, device), "gb_create: cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(GB_EUNSUPPORTED, "gb_create: device %d is sm_%d%d; libgb is built for sm_100a only",
                    device, prop.major, prop.minor);
    DeviceGuard g(device);
    if (!g.ok) return fail(GB_ECUDA, "gb_create: cudaSetDevice(%d) failed", device);
    gb_net *net = new (std::nothrow) gb_net();
    if (!net) return fail(GB_ENOMEM, "gb_create: host allocation");
    net->s = s;
    net->device = device;
    net->sm_count = prop.multiProcessorCount;
    for (int o = 0; o < gb::kNumOptions; ++o) net->opt[o].store(gb::option_default(o));
    const size_t w8b = (size_t)s.np * s.np, wbb = (size_t)s.np * s.nw * sizeof(uint32_t);
    // Wb and, behind it, the cluster unions Wu (C x C blocks, seal_kernel's companion)
    const size_t wub = 2 * (size_t)s.C * s.C * s.Wc * sizeof(uint32_t);
    void *hs = nullptr;
    if (cudaMalloc(&net->w8, w8b) != cudaSuccess || cudaMalloc(&net->wb, wbb + wub) != cudaSuccess ||
        cudaMalloc(&net->dcount, 32) != cudaSuccess ||
        cudaHostAlloc(&hs, sizeof(gb::Status), cudaHostAllocMapped) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(net->w8);
        cudaFree(net->wb);
        cudaFree(net->dcount);
        if (hs) cudaFreeHost(hs);
        delete net;
        return fail(GB_ENOMEM, "gb_create: device allocation of W (%zu bytes)", w8b + wbb);
    }
    net->hstat = static_cast<gb::Status *>(hs);
    memset(hs, 0, sizeof(gb::Status));
    void *hd = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&hd, hs, 0);
    net->hstat_dev = static_cast<gb::Status *>(hd);
    cudaMemset(net->w8, 0, w8b);
    cudaMemset(net->wb, 0, wbb + wub);
    net->wu = net->wb + (size_t)s.np * s.nw;
    net->dflag = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(net->dcount) + 8);
    cudaMemset(net->dcount, 0, 32);
    for (int i = 0; i < 3; ++i) cudaStreamCreateWithFlags(&net->stage_stream[i], cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&net->stage_event, cudaEventDisableTiming);
    for (auto &sl : net->slot_ev)
        for (auto &ev : sl) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&net->seal_event, cudaEventDisableTiming);
    // per-call scratch comes from this pool (stream-ordered); keep freed blocks for reuse
    cudaMemPoolProps pp = {};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = device;
    if (e == cudaSuccess) e = cudaMemPoolCreate(&net->pool, &pp);
    if (e == cudaSuccess) {
        uint64_t keep = ~0ull;
        e = cudaMemPoolSetAttribute(net->pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        gb_destroy(net);
        return cuda_fail(e, "gb_create: init");
    }
    gb::sos_tc_make_map(net);   // TMA descriptor of W8 for the 4-warp tensor-core SOS kernel
    *out = net;
    return GB_OK;
}

int gb_destroy(gb_net *net) {
    if (!net) return GB_OK;
    DeviceGuard g(net->device);
    cudaDeviceSynchronize();
    for (int i = 0; i < 3; ++i)
        if (net->stage_stream[i]) cudaStreamDestroy(net->stage_stream[i]);
    if (net->stage_event) cudaEventDestroy(net->stage_event);
    for (auto &sl : net->slot_ev)
        for (auto &ev : sl)
            if (ev) cudaEventDestroy(ev);
    if (net->seal_event) cudaEventDestroy(net->seal_event);
    for (auto &v : net->gvar) {
        cudaFree(v.w8g);
        if (v.ready) cudaEventDestroy(v.ready);
    }
    if (net->pool) cudaMemPoolDestroy(net->pool);
    cudaFree(net->w8);
    cudaFree(net->wb);
    cudaFree(net->dcount);   // also holds dflag
    if (net->hstat) cudaFreeHost(net->hstat);
    delete net;
    return GB_OK;
}

int gb_set_option(gb_net *net, int option, int value) {
    if (!net) return fail(GB_EINVAL, "gb_set_option: net is NULL");
    if (option < 0 || option >= gb::kNumOptions || option > GB_OPT_SOS_BITS)
        return fail(GB_EINVAL, "gb_set_option: unknown option %d", option);
    if (option == GB_OPT_HYB8_ROWS) {
        if (value != 0 && (value < 6 || value > 8))
            return fail(GB_EINVAL, "gb_set_option: value %d not 0 or 6..8", value);
    } else {
        const int lo = (option == GB_OPT_HYB8_SPLIT || option == GB_OPT_SOS_BITS) ? -1 : 0;
        if (value < lo || value > 1) return fail(GB_EINVAL, "gb_set_option: value %d outside [%d, 1]", value, lo);
    }
    net->opt[option].store(value);
    return GB_OK;
}

int gb_get_option(gb_net *net, int option, int *value) {
    if (!net || !value) return fail(GB_EINVAL, "gb_get_option: NULL argument");
    if (option < 0 || option >= gb::kNumOptions || option > GB_OPT_SOS_BITS)
        return fail(GB_EINVAL, "gb_get_option: unknown option %d", option);
    *value = net->opt[option].load();
    return GB_OK;
}

int gb_clear(gb_net *net, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_clear: net is NULL");
    DeviceGuard g(net->device);
    cudaStream_t st = (cudaStream_t)stream;
    GB_CUDA(cudaMemsetAsync(net->w8, 0, (size_t)net->s.np * net->s.np, st), "gb_clear");
    GB_CUDA(cudaMemsetAsync(net->dcount, 0, 8, st), "gb_clear");   // invalid-message count
    net->stored = 0;
    net->sealed = false;
    net->clear_epoch += 1;
    return GB_OK;
}

int gb_store(gb_net *net, const uint16_t *msgs, int64_t m, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_store: net is NULL");
    if (m < 0) return fail(GB_EINVAL, "gb_store: m = %lld < 0", (long long)m);
    if (m == 0) return GB_OK;
    if (!msgs) return fail(GB_EINVAL, "gb_store: msgs is NULL");
    DeviceGuard g(net->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int loc = where(msgs, net->device);
    if (loc < 0) return fail(GB_EINVAL, "gb_store: msgs live on another device");
    net->sealed = false;
    net->stored += m;
    if (loc == 1) {
        gb::Call cl(net, st);
        GB_CUDA(gb::launch_store(cl, msgs, m), "gb_store: launch");
        return GB_OK;
    }
    // Host messages: stage in chunks through call-private device memory (blocking).
    std::lock_guard<std::mutex> lk(net->stage_mu);
    const int64_t chunk = std::min<int64_t>(m, 1 << 20);
    const size_t row = (size_t)net->s.C * sizeof(uint16_t);
    {
        gb::Call cl(net, st);
        uint16_t *stage = cl.alloc_n<uint16_t>((size_t)chunk * net->s.C);
        if (!stage) return fail(GB_ENOMEM, "gb_store: staging buffer of %zu bytes", (size_t)chunk * row);
        for (int64_t s0 = 0; s0 < m; s0 += chunk) {
            const int64_t n = std::min(chunk, m - s0);
            GB_CUDA(cudaMemcpyAsync(stage, msgs + s0 * net->s.C, (size_t)n * row, cudaMemcpyHostToDevice, st),
                    "gb_store: H2D");
            GB_CUDA(gb::launch_store(cl, stage, n), "gb_store: launch");
        }
    }
    GB_CUDA(cudaStreamSynchronize(st), "gb_store: sync");
    return GB_OK;
}

int gb_weights(gb_net *net, uint8_t **w8, int64_t *nbytes) {
    if (!net) return fail(GB_EINVAL, "gb_weights: net is NULL");
    if (w8) {
        *w8 = net->w8;
        net->sealed = false;   // a writable W8 is out: decode needs a new gb_seal
    }
    if (nbytes) *nbytes = (int64_t)net->s.np * net->s.np;
    return GB_OK;
}

int gb_weights_view(gb_net *net, const uint8_t **w8, int64_t *nbytes) {
    if (!net) return fail(GB_EINVAL, "gb_weights_view: net is NULL");
    if (w8) *w8 = net->w8;
    if (nbytes) *nbytes = (int64_t)net->s.np * net->s.np;
    return GB_OK;
}

int gb_bits(gb_net *net, uint32_t **wb, int64_t *nbytes) {
    if (!net) return fail(GB_EINVAL, "gb_bits: net is NULL");
    if (!net->sealed) return fail(GB_ESTATE, "gb_bits: network not sealed (Wb is built by gb_seal)");
    if (wb) *wb = net->wb;
    if (nbytes) *nbytes = (int64_t)net->s.np * net->s.nw * (int64_t)sizeof(uint32_t);
    return GB_OK;
}

int gb_or_bits(gb_net *net, const uint32_t *bits, int64_t count, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_or_bits: net is NULL");
    if (count < 0) return fail(GB_EINVAL, "gb_or_bits: count = %lld < 0", (long long)count);
    if (count == 0) return GB_OK;
    if (!bits) return fail(GB_EINVAL, "gb_or_bits: bits is NULL");
    DeviceGuard g(net->device);
    if (where(bits, net->device) != 1)
        return fail(GB_EINVAL, "gb_or_bits: bits must be device memory of the handle's device");
    net->sealed = false;
    gb::Call cl(net, (cudaStream_t)stream);
    GB_CUDA(gb::launch_or_bits(cl, bits, count), "gb_or_bits: launch");
    return GB_OK;
}

int gb_or_bits_multimem(gb_net *net, const uint32_t *mc_bits, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_or_bits_multimem: net is NULL");
    if (!mc_bits) return fail(GB_EINVAL, "gb_or_bits_multimem: mc_bits is NULL");
    if ((uintptr_t)mc_bits & 3u) return fail(GB_EINVAL, "gb_or_bits_multimem: mc_bits not 4-byte aligned");
    DeviceGuard g(net->device);
    net->sealed = false;
    gb::Call cl(net, (cudaStream_t)stream);
    GB_CUDA(gb::launch_or_multimem(cl, mc_bits), "gb_or_bits_multimem: launch");
    return GB_OK;
}

int gb_pack_upper(gb_net *net, uint32_t *out, int64_t *nwords, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_pack_upper: net is NULL");
    if (nwords) *nwords = gb::upper_words(net->s);
    if (!out) return GB_OK;
    if (!net->sealed) return fail(GB_ESTATE, "gb_pack_upper: network not sealed (Wb is built by gb_seal)");
    DeviceGuard g(net->device);
    if (where(out, net->device) != 1)
        return fail(GB_EINVAL, "gb_pack_upper: out must be device memory of the handle's device");
    gb::Call cl(net, (cudaStream_t)stream);
    GB_CUDA(gb::launch_pack_upper(cl, out), "gb_pack_upper: launch");
    return GB_OK;
}

int gb_or_upper(gb_net *net, const uint32_t *sets, int64_t count, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_or_upper: net is NULL");
    if (count < 0) return fail(GB_EINVAL, "gb_or_upper: count = %lld < 0", (long long)count);
    if (count == 0) return GB_OK;
    if (!sets) return fail(GB_EINVAL, "gb_or_upper: sets is NULL");
    DeviceGuard g(net->device);
    if (where(sets, net->device) != 1)
        return fail(GB_EINVAL, "gb_or_upper: sets must be device memory of the handle's device");
    net->sealed = false;
    gb::Call cl(net, (cudaStream_t)stream);
    GB_CUDA(gb::launch_or_upper(cl, sets, count), "gb_or_upper: launch");
    return GB_OK;
}

int gb_seal(gb_net *net, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_seal: net is NULL");
    DeviceGuard g(net->device);
    cudaStream_t st = (cudaStream_t)stream;
    {
        std::lock_guard<std::mutex> lk(net->smu);
        net->seal_gen += 1;
        net->seal_epoch = net->clear_epoch;
        GB_CUDA(gb::launch_seal(net, st), "gb_seal: launch");
        GB_CUDA(cudaEventRecord(net->seal_event, st), "gb_seal: record");
    }
    net->sealed = true;
    return GB_OK;
}

int gb_seal_status(gb_net *net) {
    if (!net) return fail(GB_EINVAL, "gb_seal_status: net is NULL");
    DeviceGuard g(net->device);
    return resolve_seal(net, true);
}

int gb_decode(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma, int max_iters,
              uint32_t *out_state, uint16_t *out_iters, uint8_t *out_status, void *stream) {
    return gb_decode_ex(net, probes, k, rule, gamma, max_iters, 0u, out_state, out_iters, out_status, stream);
}

// gb_decode_ex (out_sym == nullptr: state bits into out_state) and gb_decode_symbols
// (out_state == nullptr: the state goes to call-private scratch, symbols into out_sym).
static int decode_impl(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma, int max_iters,
                       unsigned flags, uint32_t *out_state, uint16_t *out_sym, uint16_t *out_iters,
                       uint8_t *out_status, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_decode: net is NULL");
    if (flags & ~(unsigned)GB_FLAG_CYCLE_EXIT) return fail(GB_EINVAL, "gb_decode: unknown flags 0x%x", flags);
    const int cyc = (rule == GB_SUM_OF_SUM && (flags & GB_FLAG_CYCLE_EXIT)) ? 1 : 0;
    if (rule != GB_SUM_OF_SUM && rule != GB_SUM_OF_MAX && rule != GB_HYBRID)
        return fail(GB_EINVAL, "gb_decode: unknown rule %d", rule);
    if (gamma < 0 || gamma > 65535) return fail(GB_EINVAL, "gb_decode: gamma %d outside [0, 65535]", gamma);
    if (gamma == 0 && rule != GB_SUM_OF_SUM)
        return fail(GB_EINVAL, "gb_decode: sum-of-max / hybrid need gamma > 0 (Thm 1)");
    if (max_iters < 1 || max_iters > 65535)
        return fail(GB_EINVAL, "gb_decode: max_iters %d outside [1, 65535]", max_iters);
    if (k < 0) return fail(GB_EINVAL, "gb_decode: k = %lld < 0", (long long)k);
    if (!net->sealed) return fail(GB_ESTATE, "gb_decode: network not sealed (call gb_seal after gb_store)");
    DeviceGuard g(net->device);
    // the latest seal's outcome, if it has reached the host (no wait): a W that broke
    // Eq.(1)'s invariants is not decoded
    if (resolve_seal(net, false) == GB_EINVAL && net->seal_broken)
        return fail(GB_ESTATE, "gb_decode: the last gb_seal found W8 breaking Eq.(1)'s invariants (%s)",
                    net->seal_msg);
    if (k == 0) return GB_OK;
    const bool sym = out_sym != nullptr;
    void *out_main = sym ? (void *)out_sym : (void *)out_state;
    if (!probes || !out_main || !out_iters || !out_status)
        return fail(GB_EINVAL, "gb_decode: NULL buffer");
    cudaStream_t st = (cudaStream_t)stream;
    const int l0 = where(probes, net->device), l1 = where(out_main, net->device),
              l2 = where(out_iters, net->device), l3 = where(out_status, net->device);
    if (l0 < 0 || l1 < 0 || l2 < 0 || l3 < 0)
        return fail(GB_EINVAL, "gb_decode: buffer on another device");
    if (l0 && l1 && l2 && l3) {
        gb::Call cl(net, st);
        uint32_t *state = sym ? cl.alloc_n<uint32_t>((size_t)k * net->s.nw) : out_state;
        if (!state) return cuda_fail(cl.err, "gb_decode: state scratch");
        GB_CUDA(gb::launch_decode(cl, probes, k, rule, gamma, max_iters, cyc, state, out_iters, out_status),
                "gb_decode: launch");
        if (sym) GB_CUDA(gb::launch_symbols(cl, state, k, out_sym), "gb_decode_symbols: launch");
        return GB_OK;
    }
    if (l0 || l1 || l2 || l3)
        return fail(GB_EINVAL, "gb_decode: mix of host and device buffers");

    // Host buffers: a three-stage pipeline over the handle's copy-in, compute and copy-out
    // streams and kStageSlots staging slots: chunk i's H2D copy (slot i % 3, once the copy-out of
    // chunk i - 3 has left that slot), its decode (after its H2D), its D2H copies (after its
    // decode).  The two copy directions run concurrently (PCIe is full duplex) instead of
    // alternating.  Every chunk is its own call (private scratch).  Ordered after `stream`'s
    // prior work; blocks until done; host-buffer calls on one handle are serialised.
    std::lock_guard<std::mutex> lk(net->stage_mu);
    constexpr int NS = gb_net::kStageSlots;
    const size_t pin = (size_t)net->s.C * sizeof(uint16_t);
    const size_t pout = (size_t)net->s.nw * sizeof(uint32_t) + sizeof(uint16_t) + sizeof(uint8_t) +
                        (sym ? (size_t)net->s.C * sizeof(uint16_t) : 0);
    const int64_t chunk = std::min<int64_t>(k, 1 << 19);
    const size_t slot = ((size_t)chunk * (pin + pout) + 512 + 255) & ~(size_t)255;
    char *stage = nullptr;
    GB_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&stage), NS * slot, net->pool, st),
            "gb_decode: staging buffer");
    GB_CUDA(cudaEventRecord(net->stage_event, st), "gb_decode: record");
    for (int i = 0; i < 3; ++i)
        GB_CUDA(cudaStreamWaitEvent(net->stage_stream[i], net->stage_event, 0), "gb_decode: wait");
    cudaStream_t s_in = net->stage_stream[0], s_k = net->stage_stream[1], s_out = net->stage_stream[2];
    int64_t ci = 0;
    int rc = GB_OK;
    for (int64_t s0 = 0; s0 < k && rc == GB_OK; s0 += chunk, ++ci) {
        const int64_t n = std::min(chunk, k - s0);
        const int sl = (int)(ci % NS);
        cudaEvent_t *ev = net->slot_ev[sl];   // [0] copied in, [1] decoded, [2] copied out
        char *base = stage + sl * slot;
        uint16_t *dp = (uint16_t *)base;
        uint32_t *ds = (uint32_t *)(base + (((size_t)chunk * pin + 255) & ~(size_t)255));
        uint16_t *di = (uint16_t *)((char *)ds + (size_t)chunk * net->s.nw * sizeof(uint32_t));
        uint8_t *dt = (uint8_t *)(di + chunk);
        uint16_t *dy = (uint16_t *)(((uintptr_t)(dt + chunk) + 15) & ~(uintptr_t)15);   // symbols
        cudaError_t e = cudaSuccess;
        if (ci >= NS) e = cudaStreamWaitEvent(s_in, ev[2], 0);   // the slot's previous chunk has left
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(dp, probes + s0 * net->s.C, (size_t)n * pin, cudaMemcpyHostToDevice, s_in);
        if (e == cudaSuccess) e = cudaEventRecord(ev[0], s_in);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s_k, ev[0], 0);
        if (e == cudaSuccess) {
            gb::Call cl(net, s_k);
            e = gb::launch_decode(cl, dp, n, rule, gamma, max_iters, cyc, ds, di, dt);
        }
        if (e == cudaSuccess && sym) {
            gb::Call cl(net, s_k);
            e = gb::launch_symbols(cl, ds, n, dy);
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev[1], s_k);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s_out, ev[1], 0);
        if (e == cudaSuccess)
            e = sym ? cudaMemcpyAsync(out_sym + s0 * net->s.C, dy, (size_t)n * net->s.C * sizeof(uint16_t),
                                      cudaMemcpyDeviceToHost, s_out)
                    : cudaMemcpyAsync(out_state + s0 * net->s.nw, ds, (size_t)n * net->s.nw * sizeof(uint32_t),
                                      cudaMemcpyDeviceToHost, s_out);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(out_iters + s0, di, (size_t)n * sizeof(uint16_t), cudaMemcpyDeviceToHost, s_out);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out_status + s0, dt, (size_t)n, cudaMemcpyDeviceToHost, s_out);
        if (e == cudaSuccess) e = cudaEventRecord(ev[2], s_out);
        if (e != cudaSuccess) rc = cuda_fail(e, "gb_decode: staged chunk");
    }
    for (int i = 0; i < 3; ++i) {
        cudaError_t e = cudaStreamSynchronize(net->stage_stream[i]);
        if (e != cudaSuccess && rc == GB_OK) rc = cuda_fail(e, "gb_decode: sync");
    }
    cudaFreeAsync(stage, st);   // the staging streams are idle now
    return rc;
}

int gb_decode_ex(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma, int max_iters,
                 unsigned flags, uint32_t *out_state, uint16_t *out_iters, uint8_t *out_status, void *stream) {
    if (!out_state && k > 0) return fail(GB_EINVAL, "gb_decode: NULL buffer");
    return decode_impl(net, probes, k, rule, gamma, max_iters, flags, out_state, nullptr, out_iters, out_status,
                       stream);
}

int gb_decode_symbols(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma, int max_iters,
                      unsigned flags, uint16_t *out_symbols, uint16_t *out_iters, uint8_t *out_status,
                      void *stream) {
    if (!out_symbols && k > 0) return fail(GB_EINVAL, "gb_decode_symbols: NULL buffer");
    return decode_impl(net, probes, k, rule, gamma, max_iters, flags, nullptr, out_symbols, out_iters, out_status,
                       stream);
}

int gb_info(gb_net *net, int *c, int *l, int *n_padded, int64_t *stored_count) {
    if (!net) return fail(GB_EINVAL, "gb_info: net is NULL");
    if (c) *c = net->s.C;
    if (l) *l = net->s.L;
    if (n_padded) *n_padded = net->s.np;
    if (stored_count) *stored_count = net->stored;
    return GB_OK;
}

const char *gb_decode_kernel(gb_net *net, int rule) {
    if (!net) return "";
    if (rule == GB_SUM_OF_SUM && gb::sos_bits_chosen(net, 0, 0)) return "sos_bits_kernel";
    if (rule == GB_SUM_OF_SUM && gb::sos_tc3_enabled(net))
        return gb::sos_tc3_pair(net) ? "sos_tc3x2_kernel" : "sos_tc3_kernel";
    if (rule == GB_SUM_OF_SUM && gb::sos_tc2_supported(net->s))
        return gb::sos_2cta_enabled(net) ? "sos_tc2x2_kernel" : "sos_tc2_kernel";
    if (rule == GB_SUM_OF_SUM && net->wmap_ok && gb::sos_tc_supported(net->s)) return "sos_tc_kernel";
    if (rule == GB_SUM_OF_MAX && gb::som_tc_enabled(net)) return "som_tc_kernel";
    if (rule == GB_HYBRID && gb::decode_hyb8_supported(net, rule, 0, nullptr))
        return gb::decode_hyb8_rotated(net) ? "decode_hyb8r_kernel" : "decode_hyb8_kernel";
    if (rule != GB_SUM_OF_SUM && gb::decode_smem_supported(net->s, rule)) return "decode_smem_kernel";
    if (rule != GB_SUM_OF_SUM && gb::decode_l2_supported(net->s, rule))
        return gb::decode_l2t_supported(net, rule) ? "decode_l2t_kernel" : "decode_l2_kernel";
    return "decode_generic_kernel";
}

int gb_launch_count(gb_net *net, int64_t *launches) {
    if (!net || !launches) return fail(GB_EINVAL, "gb_launch_count: NULL argument");
    *launches = net->launches.load();
    return GB_OK;
}

}  // extern "C"

namespace gb {

int option_default(int o) {
    switch (o) {
        case kOptSosPair: return 1;
        case kOptSosStreamed: return 1;
        case kOptSomTensor: return 0;
        case kOptHyb8: return 1;
        case kOptL2t: return 1;
        case kOptHyb8Split: return -1;
        case kOptStoreScatter: return 0;
        case kOptSosBits: return -1;
        default: return 0;
    }
}

Call::~Call() {
    for (int i = nblk_ - 1; i >= 0; --i) cudaFreeAsync(blk_[i], st);
}

void *Call::alloc(size_t bytes) {
    if (nblk_ == 8) {
        err = cudaErrorMemoryAllocation;
        return nullptr;
    }
    void *p = nullptr;
    cudaError_t e = cudaMallocFromPoolAsync(&p, bytes ? bytes : 16, net->pool, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        err = cudaErrorMemoryAllocation;
        return nullptr;
    }
    blk_[nblk_++] = p;
    return p;
}

unsigned long long *Call::counters() {
    if (!counters_) {
        counters_ = alloc_n<unsigned long long>(3);
        if (!counters_) return nullptr;
        cudaError_t e = cudaMemsetAsync(counters_, 0, 3 * sizeof(unsigned long long), st);
        if (e != cudaSuccess) {
            err = e;
            counters_ = nullptr;
        }
    }
    return counters_;
}

int64_t *Call::ovf(int64_t k) {
    if (!ovf_) ovf_ = alloc_n<int64_t>((size_t)(k > 0 ? k : 1));
    return ovf_;
}

// W density below which sum-of-sum runs on the CUDA cores (gb_decode_sos_bits.cu).  Measured
// crossover (c=8 l=128 e=4, 10^6 probes, sos_bits vs sos_tc2x2 ms): M=3k (d=0.17) 0.52 vs 1.92,
// M=5k (0.26) 0.95 vs 2.51, M=8k (0.39) 2.10 vs 3.45, M=10k (0.46) 3.65 vs 3.80, M=12k (0.52)
// 5.08 vs 4.03.
constexpr double kSosBitsDensity = 0.45;

bool sos_bits_chosen(const gb_net *net, int gamma, int cyc) {
    const int ob = net->opt[kOptSosBits].load(std::memory_order_relaxed);
    return sos_bits_supported(net->s, gamma, cyc) &&
           (ob == 1 || (ob < 0 && net->density.load(std::memory_order_relaxed) < kSosBitsDensity));
}

// Kernel selection for one decode call.
cudaError_t launch_decode(Call &cl, const uint16_t *probes, int64_t k, int rule, int gamma, int max_iters, int cyc,
                          uint32_t *state, uint16_t *iters, uint8_t *status) {
    gb_net *net = cl.net;
    cudaError_t e = cudaErrorNotSupported;
    if (rule == GB_SUM_OF_SUM) {
        // sparse states (low W density): active rows into bit-sliced counters on the CUDA cores
        if (sos_bits_chosen(net, gamma, cyc))
            e = launch_sos_bits(cl, probes, k, gamma, max_iters, state, iters, status);
        else if (sos_tc2_supported(net->s) || sos_tc3_enabled(net) || (net->wmap_ok && sos_tc_supported(net->s)))
            e = launch_decode_sos_tc(cl, probes, k, gamma, max_iters, cyc, state, iters, status);
    } else {
        if (rule == GB_SUM_OF_MAX && som_tc_enabled(net))
            e = launch_som_tc(cl, probes, k, max_iters, state, iters, status);
        if (e == cudaErrorNotSupported) e = launch_decode_smem(cl, probes, k, rule, max_iters, state, iters, status);
        if (e == cudaErrorNotSupported) e = launch_decode_l2(cl, probes, k, rule, max_iters, state, iters, status);
    }
    if (e != cudaErrorNotSupported) return e;
    return launch_decode_generic(cl, probes, k, rule, gamma, max_iters, cyc, state, iters, status);
}

}  // namespace gb
