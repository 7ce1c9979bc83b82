// gb_api.cu -- the C-ABI of libgb (include/gb.h): handle lifecycle,
// argument validation, error reporting, host-buffer staging and dispatch to
// the sm_100a kernels.  No compute happens on the host: every step of
// store/seal/decode runs in the kernels of gb_store.cu / gb_decode_*.cu.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "gb_internal.h"

namespace gb {
cudaError_t launch_decode_smem(gb_net *net, const uint16_t *probes, int64_t k, int rule, int max_iters,
                               uint32_t *state, uint16_t *iters, uint8_t *status, cudaStream_t st);
cudaError_t launch_decode_generic(gb_net *net, const uint16_t *probes, int64_t k, int rule,
                                  int gamma, int max_iters, int cyc, uint32_t *state, uint16_t *iters,
                                  uint8_t *status, cudaStream_t st);
}

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

int ensure_stage(gb_net *net, size_t bytes) {
    if (net->stage_bytes >= bytes) return GB_OK;
    if (net->stage) cudaFree(net->stage);
    net->stage = nullptr;
    net->stage_bytes = 0;
    if (cudaMalloc(&net->stage, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(GB_ENOMEM, "staging buffer of %zu bytes", bytes);
    }
    net->stage_bytes = bytes;
    return GB_OK;
}

}  // namespace

extern "C" {

const char *gb_last_error(void) { return g_err; }

const char *gb_version(void) { return "libgb 0.1 (sm_100a)"; }

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
    gb_net *net = (gb_net *)calloc(1, sizeof(gb_net));
    if (!net) return fail(GB_ENOMEM, "gb_create: host allocation");
    net->s = s;
    net->device = device;
    net->sm_count = prop.multiProcessorCount;
    const size_t w8b = (size_t)s.np * s.np, wbb = (size_t)s.np * s.nw * sizeof(uint32_t);
    if (cudaMalloc(&net->w8, w8b) != cudaSuccess || cudaMalloc(&net->wb, wbb) != cudaSuccess ||
        cudaMalloc(&net->dcount, 16) != cudaSuccess ||   // [0, 8) invalid-message count, [8, 12) flags
        cudaMallocHost(&net->hstat, 16) != cudaSuccess ||
        cudaMalloc(&net->queue, sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&net->ovf_count, sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(net->w8); cudaFree(net->wb); cudaFree(net->dcount); cudaFreeHost(net->hstat); cudaFree(net->queue); cudaFree(net->ovf_count);
        free(net);
        return fail(GB_ENOMEM, "gb_create: device allocation of W (%zu bytes)", w8b + wbb);
    }
    cudaMemset(net->w8, 0, w8b);
    cudaMemset(net->wb, 0, wbb);
    net->dflag = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(net->dcount) + 8);
    cudaMemset(net->dcount, 0, 16);
    for (int i = 0; i < 2; ++i) cudaStreamCreateWithFlags(&net->stage_stream[i], cudaStreamNonBlocking);
    for (int i = 0; i < 4; ++i) cudaEventCreateWithFlags(&net->stage_event[i], cudaEventDisableTiming);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        gb_destroy(net);
        return cuda_fail(e, "gb_create: init");
    }
    gb::sos_tc_make_map(net);   // TMA descriptor of W8 for the tensor-core SOS kernel
    *out = net;
    return GB_OK;
}

int gb_destroy(gb_net *net) {
    if (!net) return GB_OK;
    DeviceGuard g(net->device);
    cudaDeviceSynchronize();
    for (int i = 0; i < 2; ++i) if (net->stage_stream[i]) cudaStreamDestroy(net->stage_stream[i]);
    for (int i = 0; i < 4; ++i) if (net->stage_event[i]) cudaEventDestroy(net->stage_event[i]);
    cudaFree(net->stage);
    cudaFree(net->w8g);
    cudaFree(net->vscratch);
    cudaFree(net->w8);
    cudaFree(net->wb);
    cudaFree(net->dcount);   // also holds dflag
    cudaFreeHost(net->hstat);
    cudaFree(net->queue);
    cudaFree(net->ovf);
    cudaFree(net->ovf_count);
    cudaFree(net->spart);
    cudaFree(net->xscratch);
    cudaFree(net->w4);
    free(net);
    return GB_OK;
}

int gb_clear(gb_net *net, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_clear: net is NULL");
    DeviceGuard g(net->device);
    cudaStream_t st = (cudaStream_t)stream;
    GB_CUDA(cudaMemsetAsync(net->w8, 0, (size_t)net->s.np * net->s.np, st), "gb_clear");
    GB_CUDA(cudaMemsetAsync(net->dcount, 0, 16, st), "gb_clear");   // count + flags
    net->stored = 0;
    net->sealed = false;
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
        GB_CUDA(gb::launch_store(net, msgs, m, st), "gb_store: launch");
        return GB_OK;
    }
    // Host messages: stage in chunks through device scratch (blocking).
    const int64_t chunk = std::min<int64_t>(m, 1 << 20);
    const size_t row = (size_t)net->s.C * sizeof(uint16_t);
    int rc = ensure_stage(net, (size_t)chunk * row);
    if (rc) return rc;
    for (int64_t s0 = 0; s0 < m; s0 += chunk) {
        const int64_t n = std::min(chunk, m - s0);
        GB_CUDA(cudaMemcpyAsync(net->stage, msgs + s0 * net->s.C, (size_t)n * row,
                                cudaMemcpyHostToDevice, st), "gb_store: H2D");
        GB_CUDA(gb::launch_store(net, (const uint16_t *)net->stage, n, st), "gb_store: launch");
    }
    GB_CUDA(cudaStreamSynchronize(st), "gb_store: sync");
    return GB_OK;
}

int gb_weights(gb_net *net, uint8_t **w8, int64_t *nbytes) {
    if (!net) return fail(GB_EINVAL, "gb_weights: net is NULL");
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
    if (where(bits, net->device) != 1) return fail(GB_EINVAL, "gb_or_bits: bits must be device memory of the handle's device");
    net->sealed = false;
    GB_CUDA(gb::launch_or_bits(net, bits, count, (cudaStream_t)stream), "gb_or_bits: launch");
    return GB_OK;
}

int gb_seal(gb_net *net, void *stream) {
    if (!net) return fail(GB_EINVAL, "gb_seal: net is NULL");
    DeviceGuard g(net->device);
    cudaStream_t st = (cudaStream_t)stream;
    GB_CUDA(gb::launch_seal(net, st), "gb_seal: launch");
    net->launches += 1;
    unsigned flag = 0;
    unsigned long long cnt = 0;
    // count and flags in one 16-byte copy to pinned memory, then one reset
    GB_CUDA(cudaMemcpyAsync(net->hstat, net->dcount, 16, cudaMemcpyDeviceToHost, st), "gb_seal: status");
    GB_CUDA(cudaStreamSynchronize(st), "gb_seal: sync");
    memcpy(&cnt, net->hstat, sizeof cnt);
    memcpy(&flag, reinterpret_cast<const char *>(net->hstat) + 8, sizeof flag);
    unsigned edges = 0;
    memcpy(&edges, reinterpret_cast<const char *>(net->hstat) + 12, sizeof edges);
    {
        const double pairs = (double)net->s.C * (net->s.C - 1) * (double)net->s.L * net->s.L;
        net->density = pairs > 0 ? edges / pairs : 0.0;
    }
    GB_CUDA(cudaMemsetAsync(net->dcount, 0, 16, st), "gb_seal: reset");
    const unsigned structural = flag & ~gb::kFlagStoreInvalid;
    if (structural) {
        net->sealed = false;
        return fail(GB_EINVAL, "gb_seal: W8 breaks Eq.(1) invariants:%s%s%s%s",
                    (structural & gb::kFlagNotBinary) ? " non-binary entry" : "",
                    (structural & gb::kFlagAsym) ? " asymmetric" : "",
                    (structural & gb::kFlagIntra) ? " intra-cluster edge" : "",
                    (structural & gb::kFlagPad) ? " padding edge" : "");
    }
    net->sealed = true;
    net->seal_gen += 1;
    if (cnt) return fail(GB_EINVAL, "gb_seal: %llu stored message(s) had a symbol >= L and were skipped",
                         (unsigned long long)cnt);
    return GB_OK;
}

int gb_decode(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma, int max_iters,
              uint32_t *out_state, uint16_t *out_iters, uint8_t *out_status, void *stream) {
    return gb_decode_ex(net, probes, k, rule, gamma, max_iters, 0u, out_state, out_iters, out_status, stream);
}

int gb_decode_ex(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma, int max_iters,
                 unsigned flags, uint32_t *out_state, uint16_t *out_iters, uint8_t *out_status, void *stream) {
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
    if (k == 0) return GB_OK;
    if (!probes || !out_state || !out_iters || !out_status)
        return fail(GB_EINVAL, "gb_decode: NULL buffer");
    DeviceGuard g(net->device);
    cudaStream_t st = (cudaStream_t)stream;
    const int l0 = where(probes, net->device), l1 = where(out_state, net->device),
              l2 = where(out_iters, net->device), l3 = where(out_status, net->device);
    if (l0 < 0 || l1 < 0 || l2 < 0 || l3 < 0)
        return fail(GB_EINVAL, "gb_decode: buffer on another device");
    if (l0 && l1 && l2 && l3) {
        GB_CUDA(gb::launch_decode(net, probes, k, rule, gamma, max_iters, cyc, out_state, out_iters,
                                  out_status, st),
                "gb_decode: launch");
        return GB_OK;
    }
    if (l0 || l1 || l2 || l3)
        return fail(GB_EINVAL, "gb_decode: mix of host and device buffers");

    // Host buffers: double-buffered pipeline over two library streams;
    // chunk i: H2D probes -> decode -> D2H results, overlapping with chunk
    // i+1's copies.  Ordered after `stream`'s prior work; blocks until done.
    const size_t pin = (size_t)net->s.C * sizeof(uint16_t);
    const size_t pout = (size_t)net->s.nw * sizeof(uint32_t) + sizeof(uint16_t) + sizeof(uint8_t);
    const int64_t chunk = std::min<int64_t>(k, 1 << 19);
    const size_t slot = ((size_t)chunk * (pin + pout) + 255) & ~(size_t)255;
    int rc = ensure_stage(net, 2 * slot);
    if (rc) return rc;
    GB_CUDA(cudaEventRecord(net->stage_event[2], st), "gb_decode: record");
    for (int i = 0; i < 2; ++i)
        GB_CUDA(cudaStreamWaitEvent(net->stage_stream[i], net->stage_event[2], 0), "gb_decode: wait");
    int64_t ci = 0;
    for (int64_t s0 = 0; s0 < k; s0 += chunk, ++ci) {
        const int64_t n = std::min(chunk, k - s0);
        const int sl = (int)(ci & 1);
        cudaStream_t ss = net->stage_stream[sl];
        char *base = (char *)net->stage + sl * slot;
        uint16_t *dp = (uint16_t *)base;
        uint32_t *ds = (uint32_t *)(base + (((size_t)chunk * pin + 255) & ~(size_t)255));
        uint16_t *di = (uint16_t *)((char *)ds + (size_t)chunk * net->s.nw * sizeof(uint32_t));
        uint8_t *dt = (uint8_t *)(di + chunk);
        GB_CUDA(cudaMemcpyAsync(dp, probes + s0 * net->s.C, (size_t)n * pin, cudaMemcpyHostToDevice, ss),
                "gb_decode: H2D");
        GB_CUDA(gb::launch_decode(net, dp, n, rule, gamma, max_iters, cyc, ds, di, dt, ss), "gb_decode: launch");
        GB_CUDA(cudaMemcpyAsync(out_state + s0 * net->s.nw, ds, (size_t)n * net->s.nw * sizeof(uint32_t),
                                cudaMemcpyDeviceToHost, ss), "gb_decode: D2H state");
        GB_CUDA(cudaMemcpyAsync(out_iters + s0, di, (size_t)n * sizeof(uint16_t), cudaMemcpyDeviceToHost, ss),
                "gb_decode: D2H iters");
        GB_CUDA(cudaMemcpyAsync(out_status + s0, dt, (size_t)n, cudaMemcpyDeviceToHost, ss),
                "gb_decode: D2H status");
    }
    for (int i = 0; i < 2; ++i) GB_CUDA(cudaStreamSynchronize(net->stage_stream[i]), "gb_decode: sync");
    return GB_OK;
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
    if (rule == GB_SUM_OF_SUM && gb::sos_fp4_enabled(net->s, 2)) return "sos_fp4_kernel";   // (gamma = 2)
    if (rule == GB_SUM_OF_SUM && gb::sos_tc2_supported(net->s))
        return gb::sos_2cta_enabled(net->s) ? "sos_tc2x2_kernel" : "sos_tc2_kernel";
    if (rule == GB_SUM_OF_SUM && gb::sos_tc3_enabled(net->s))
        return gb::sos_tc3_pair(net->s) ? "sos_tc3x2_kernel" : "sos_tc3_kernel";
    if (rule == GB_SUM_OF_SUM && net->wmap_ok && gb::sos_tc_supported(net->s)) return "sos_tc_kernel";
    if (rule == GB_SUM_OF_MAX && gb::som_tc_enabled(net->s)) return "som_tc_kernel";
    if (rule == GB_HYBRID && gb::decode_hyb8_supported(net->s, rule, 0, nullptr)) return "decode_hyb8_kernel";
    if (rule != GB_SUM_OF_SUM && gb::decode_smem_supported(net->s, rule)) return "decode_smem_kernel";
    if (rule != GB_SUM_OF_SUM && gb::decode_l2_supported(net->s, rule))
        return gb::decode_l2t_supported(net->s, rule) ? "decode_l2t_kernel" : "decode_l2_kernel";
    return "decode_generic_kernel";
}

int gb_launch_count(gb_net *net, int64_t *launches) {
    if (!net || !launches) return fail(GB_EINVAL, "gb_launch_count: NULL argument");
    *launches = net->launches;
    return GB_OK;
}

}  // extern "C"

namespace gb {

// Kernel selection for one decode call.
cudaError_t launch_decode(gb_net *net, const uint16_t *probes, int64_t k, int rule, int gamma,
                          int max_iters, int cyc, uint32_t *state, uint16_t *iters, uint8_t *status,
                          cudaStream_t st) {
    cudaError_t e = cudaErrorNotSupported;
    if (rule == GB_SUM_OF_SUM) {
        if (sos_tc2_supported(net->s) || sos_tc3_enabled(net->s) || (net->wmap_ok && sos_tc_supported(net->s)))
            e = launch_decode_sos_tc(net, probes, k, gamma, max_iters, cyc, state, iters, status, st);
    } else {
        if (rule == GB_SUM_OF_MAX && som_tc_enabled(net->s))
            e = launch_som_tc(net, probes, k, max_iters, state, iters, status, st);
        if (e == cudaErrorNotSupported) e = launch_decode_smem(net, probes, k, rule, max_iters, state, iters, status, st);
        if (e == cudaErrorNotSupported) e = launch_decode_l2(net, probes, k, rule, max_iters, state, iters, status, st);
    }
    if (e != cudaErrorNotSupported) return e;
    return launch_decode_generic(net, probes, k, rule, gamma, max_iters, cyc, state, iters, status, st);
}

}  // namespace gb
