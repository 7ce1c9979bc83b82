"""paper_1303_7032_b200 -- GBNN batched retrieval on B200 (arXiv:1303.7032).

Thin Python binding over the C-ABI of ``libgb.so`` (include/gb.h).  This file
only marshals arguments (pointers, sizes, the current CUDA stream); every step
of store / seal / decode runs in the sm_100a kernels behind the ABI.  There is
no CPU fallback: if ``libgb.so`` is missing or cannot load, importing
``paper_1303_7032_b200.lib`` raises, and every call needs a B200.

    net = Net(c=8, l=128)               # gb_create
    net.store(msgs)                     # gb_store  (uint16 [M, C], host or cuda)
    net.seal()                          # gb_seal
    state, iters, status = net.decode(probes, HYBRID)   # gb_decode
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

SUM_OF_SUM, SUM_OF_MAX, HYBRID = 0, 1, 2
SOS, SOM = SUM_OF_SUM, SUM_OF_MAX
CONVERGED, MAX_ITERS, INVALID, CYCLE = 0, 1, 2, 3
FLAG_CYCLE_EXIT = 1   # gb_decode_ex: stop an oscillating sum-of-sum probe at V^r == V^{r-2}
ERASED, AMBIGUOUS = 0xFFFF, 0xFFFE   # gb_decode_symbols: no / several active neurons in a cluster
ERASED = 0xFFFF
GB_OK, GB_EINVAL, GB_ENOMEM, GB_ECUDA, GB_ESTATE, GB_EUNSUPPORTED = 0, -1, -2, -3, -4, -5

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GB_LIB", os.path.join(_HERE, "libgb.so"))   # GB_LIB: experiment builds

# Every symbol include/gb.h declares (checked by tests/test_abi.py).
EXPORTS = ("gb_create", "gb_destroy", "gb_clear", "gb_store", "gb_set_option", "gb_get_option", "gb_weights",
           "gb_or_bits_multimem",
           "gb_weights_view", "gb_bits", "gb_or_bits", "gb_pack_upper", "gb_or_upper", "gb_seal", "gb_seal_status",
           "gb_decode", "gb_decode_ex", "gb_decode_symbols", "gb_info",
           "gb_launch_count", "gb_decode_kernel", "gb_last_error", "gb_version")

# gb_set_option keys (include/gb.h GB_OPT_*): kernel choices with identical results
OPTIONS = {"sos_pair": 0, "sos_streamed": 1, "som_tensor": 2, "hyb8": 3, "l2t": 4, "hyb8_split": 5,
           "store_scatter": 6, "hyb8_rows": 7,
           "sos_bits": 8}

_lib = None


class GBError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def lib() -> ctypes.CDLL:
    """Load libgb.so (build it first with ``paper_1303_7032_b200.build``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "gb_create": ([i32, i32, i32, PP], i32),
        "gb_destroy": ([P], i32),
        "gb_clear": ([P, P], i32),
        "gb_store": ([P, P, i64, P], i32),
        "gb_weights": ([P, PP, ctypes.POINTER(i64)], i32),
        "gb_weights_view": ([P, PP, ctypes.POINTER(i64)], i32),
        "gb_seal": ([P, P], i32),
        "gb_seal_status": ([P], i32),
        "gb_set_option": ([P, i32, i32], i32),
        "gb_get_option": ([P, i32, ctypes.POINTER(i32)], i32),
        "gb_bits": ([P, PP, ctypes.POINTER(i64)], i32),
        "gb_or_bits": ([P, P, i64, P], i32),
        "gb_or_bits_multimem": ([P, P, P], i32),
        "gb_pack_upper": ([P, P, ctypes.POINTER(i64), P], i32),
        "gb_or_upper": ([P, P, i64, P], i32),
        "gb_decode": ([P, P, i64, i32, i32, i32, P, P, P, P], i32),
        "gb_decode_ex": ([P, P, i64, i32, i32, i32, ctypes.c_uint, P, P, P, P], i32),
        "gb_decode_symbols": ([P, P, i64, i32, i32, i32, ctypes.c_uint, P, P, P, P], i32),
        "gb_info": ([P, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32),
                     ctypes.POINTER(i64)], i32),
        "gb_launch_count": ([P, ctypes.POINTER(i64)], i32),
        "gb_decode_kernel": ([P, i32], ctypes.c_char_p),
        "gb_last_error": ([], ctypes.c_char_p),
        "gb_version": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        if "GB_LIB" in os.environ and not hasattr(L, name):
            continue   # an older experiment build (tools/ab.sh) without a newer entry point
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def _check(rc: int):
    if rc != GB_OK:
        raise GBError(rc, lib().gb_last_error().decode())
    return rc


def _stream(stream):
    if stream is None:
        import torch
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        return ctypes.c_void_p(0)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _addr(x) -> int:
    """Raw pointer of a torch tensor (host or cuda) or numpy array."""
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous
        return x.ctypes.data
    assert x.is_contiguous()
    return x.data_ptr()


class _CudaArray:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class Net:
    """One GBNN network on one CUDA device (gb_net handle).

    ``options``: kernel-selection options (``OPTIONS`` keys -> 0/1, ``hyb8_split``
    also -1, ``hyb8_rows`` 0 or 6..8), passed to gb_set_option; they pick between
    bit-exact kernels."""

    def __init__(self, c: int, l: int, device: int = 0, **options):
        h = ctypes.c_void_p()
        _check(lib().gb_create(c, l, device, ctypes.byref(h)))
        self._h = h
        self.c, self.l, self.device = c, l, device
        self.wc = (l + 31) // 32
        self.n_padded = c * 32 * self.wc
        self.nw = c * self.wc
        for k, v in options.items():
            self.set_option(k, v)

    def set_option(self, name, value: int):
        _check(lib().gb_set_option(self._h, OPTIONS[name] if isinstance(name, str) else int(name), int(value)))

    def option(self, name) -> int:
        v = ctypes.c_int()
        _check(lib().gb_get_option(self._h, OPTIONS[name] if isinstance(name, str) else int(name), ctypes.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "_h", None):
            lib().gb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def clear(self, stream=None):
        _check(lib().gb_clear(self._h, _stream(stream)))

    def store(self, msgs, stream=None):
        m = int(msgs.shape[0]) if msgs.ndim == 2 else 0
        assert msgs.ndim == 2 and msgs.shape[1] == self.c
        _check(lib().gb_store(self._h, ctypes.c_void_p(_addr(msgs)), m, _stream(stream)))

    def seal(self, stream=None, check: bool = True):
        """gb_seal (asynchronous); with ``check`` also gb_seal_status (waits for it and
        raises GBError on broken invariants or skipped invalid messages)."""
        _check(lib().gb_seal(self._h, _stream(stream)))
        if check:
            self.seal_status()

    def seal_status(self):
        _check(lib().gb_seal_status(self._h))

    def weights(self):
        """The library-owned W8 as a torch uint8 cuda tensor [n_p, n_p] (no copy).
        Unseals the net (it may be written): call seal() before decoding."""
        import torch
        p = ctypes.c_void_p()
        nb = ctypes.c_int64()
        _check(lib().gb_weights(self._h, ctypes.byref(p), ctypes.byref(nb)))
        arr = _CudaArray(p.value, (self.n_padded, self.n_padded), "|u1")
        return torch.as_tensor(arr, device=f"cuda:{self.device}")

    def weights_view(self):
        """W8 for reading only (gb_weights_view): the net stays sealed; do not write it."""
        import torch
        p = ctypes.c_void_p()
        nb = ctypes.c_int64()
        _check(lib().gb_weights_view(self._h, ctypes.byref(p), ctypes.byref(nb)))
        arr = _CudaArray(p.value, (self.n_padded, self.n_padded), "|u1")
        return torch.as_tensor(arr, device=f"cuda:{self.device}")

    def bits(self):
        """The library-owned packed rows Wb as a torch int32 cuda tensor [n_p, nw]
        (no copy; valid after seal until W changes)."""
        import torch
        p = ctypes.c_void_p()
        nb = ctypes.c_int64()
        _check(lib().gb_bits(self._h, ctypes.byref(p), ctypes.byref(nb)))
        arr = _CudaArray(p.value, (self.n_padded, self.nw), "<i4")
        return torch.as_tensor(arr, device=f"cuda:{self.device}")

    def or_bits(self, bits, stream=None):
        """gb_or_bits: OR packed bit matrices ([count, n_p, nw] int32 cuda tensor) into W8."""
        assert bits.is_cuda and bits.is_contiguous() and tuple(bits.shape[-2:]) == (self.n_padded, self.nw)
        count = bits.numel() // (self.n_padded * self.nw)
        _check(lib().gb_or_bits(self._h, ctypes.c_void_p(bits.data_ptr()), count, _stream(stream)))

    def or_bits_multimem(self, mc_ptr: int, stream=None):
        """gb_or_bits_multimem: OR into W8 the packed matrices every GPU of a multicast group
        holds at the multicast address mc_ptr (NVLS reduction, one multimem.ld_reduce.or per word)."""
        _check(lib().gb_or_bits_multimem(self._h, ctypes.c_void_p(mc_ptr), _stream(stream)))

    def upper_words(self) -> int:
        n = ctypes.c_int64()
        _check(lib().gb_pack_upper(self._h, None, ctypes.byref(n), None))
        return n.value

    def pack_upper(self, out=None, stream=None):
        """gb_pack_upper: the upper-triangle blocks of the sealed Wb as an int32 cuda tensor."""
        import torch
        n = self.upper_words()
        if out is None:
            out = torch.empty((n,), dtype=torch.int32, device=f"cuda:{self.device}")
        assert out.is_cuda and out.is_contiguous() and out.numel() == n
        _check(lib().gb_pack_upper(self._h, ctypes.c_void_p(out.data_ptr()), None, _stream(stream)))
        return out

    def or_upper(self, sets, stream=None):
        """gb_or_upper: OR packed upper-triangle sets ([count, n] int32 cuda tensor) into W8."""
        n = self.upper_words()
        assert sets.is_cuda and sets.is_contiguous() and sets.numel() % n == 0
        _check(lib().gb_or_upper(self._h, ctypes.c_void_p(sets.data_ptr()), sets.numel() // n, _stream(stream)))

    def info(self):
        c, l, n, s = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _check(lib().gb_info(self._h, ctypes.byref(c), ctypes.byref(l), ctypes.byref(n),
                             ctypes.byref(s)))
        return c.value, l.value, n.value, s.value

    def launch_count(self) -> int:
        n = ctypes.c_int64()
        _check(lib().gb_launch_count(self._h, ctypes.byref(n)))
        return n.value

    def decode_kernel(self, rule: int) -> str:
        return lib().gb_decode_kernel(self._h, rule).decode()

    def alloc_outputs(self, k: int, device: bool = True, pin: bool = False):
        import torch
        kw = dict(device=f"cuda:{self.device}") if device else dict(pin_memory=pin)
        state = torch.empty((k, self.nw), dtype=torch.int32, **kw)
        iters = torch.empty((k,), dtype=torch.int16, **kw)
        status = torch.empty((k,), dtype=torch.uint8, **kw)
        return state, iters, status

    def decode(self, probes, rule: int, gamma: int = 2, max_iters: int = 20, out=None,
               stream=None, flags: int = 0):
        """gb_decode.  ``probes``: uint16-bit [K, C] torch tensor (cuda or host)
        or numpy array.  Returns (state int32 [K, nw], iters int16 [K],
        status uint8 [K]) on the probes' side (bit patterns; view as unsigned)."""
        k = int(probes.shape[0])
        assert probes.ndim == 2 and probes.shape[1] == self.c
        if out is None:
            if isinstance(probes, np.ndarray):
                out = (np.empty((k, self.nw), np.uint32), np.empty(k, np.uint16),
                       np.empty(k, np.uint8))
            else:
                out = self.alloc_outputs(k, device=probes.is_cuda)
        state, iters, status = out
        _check(lib().gb_decode_ex(self._h, ctypes.c_void_p(_addr(probes)), k, rule, gamma, max_iters, flags,
                                  ctypes.c_void_p(_addr(state)), ctypes.c_void_p(_addr(iters)),
                                  ctypes.c_void_p(_addr(status)), _stream(stream)))
        return state, iters, status

    def decode_symbols(self, probes, rule: int, gamma: int = 2, max_iters: int = 20, out=None,
                       stream=None, flags: int = 0):
        """gb_decode_symbols: the retrieved message instead of the state bits.  Returns
        (symbols int16 [K, C] (bit patterns of uint16: l, ERASED or AMBIGUOUS), iters int16 [K],
        status uint8 [K]) on the probes' side."""
        k = int(probes.shape[0])
        assert probes.ndim == 2 and probes.shape[1] == self.c
        if out is None:
            if isinstance(probes, np.ndarray):
                out = (np.empty((k, self.c), np.uint16), np.empty(k, np.uint16), np.empty(k, np.uint8))
            else:
                import torch
                dev = probes.device
                pin = not probes.is_cuda
                out = (torch.empty((k, self.c), dtype=torch.int16, device=dev, pin_memory=pin),
                       torch.empty(k, dtype=torch.int16, device=dev, pin_memory=pin),
                       torch.empty(k, dtype=torch.uint8, device=dev, pin_memory=pin))
        sym, iters, status = out
        _check(lib().gb_decode_symbols(self._h, ctypes.c_void_p(_addr(probes)), k, rule, gamma, max_iters, flags,
                                       ctypes.c_void_p(_addr(sym)), ctypes.c_void_p(_addr(iters)),
                                       ctypes.c_void_p(_addr(status)), _stream(stream)))
        return sym, iters, status
