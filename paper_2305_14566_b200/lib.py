"""ctypes binding of libomniseg.so (include/omniseg.h, include/omniseg_debug.h).

Argument marshalling only: every step of the path runs in the library's CUDA
kernels. There is no fallback -- if the in-tree library is missing or cannot
be loaded, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OMNISEG_LIB", os.path.join(HERE, "lib", "libomniseg.so"))

_lib = None

# Every symbol include/omniseg.h and include/omniseg_debug.h declare.
SYMBOLS = ("omniseg_create", "omniseg_segment_slide", "omniseg_output_size", "omniseg_comm_init",
           "omniseg_segment_band", "omniseg_gather_bands", "omniseg_band_rows", "omniseg_render_overlay", "omniseg_get_tiles",
           "omniseg_get_fgmask",
           "omniseg_get_timings", "omniseg_set_stream", "omniseg_last_error", "omniseg_destroy",
           "omniseg_debug_predict_tiles", "omniseg_debug_conv", "omniseg_debug_set_profile",
           "omniseg_debug_get_profile", "omniseg_debug_band_globals", "omniseg_debug_band_fg", "omniseg_debug_get_detection")


class OmnisegError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"omniseg error {code}: {msg}")
        self.code = code


def load(path: str = LIB_PATH):
    """Load (once) and return the library with argtypes set. Raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OmnisegError(-2, f"{path} not found: run `python -m paper_2305_14566_b200.build` "
                               "(there is no CPU fallback)")
    L = C.CDLL(path)
    vp, i64, i32, sz = C.c_void_p, C.c_int64, C.c_int, C.c_size_t
    L.omniseg_create.argtypes = [C.c_char_p, vp, sz]
    L.omniseg_create.restype = vp
    L.omniseg_segment_slide.argtypes = [vp, vp, i64, i64, i32, i32, i32, vp, vp, i32, vp, vp, vp]
    L.omniseg_segment_slide.restype = i32
    L.omniseg_output_size.argtypes = [vp, i64, i64, i32]
    L.omniseg_output_size.restype = i64
    L.omniseg_comm_init.argtypes = [vp, vp, i32, i32]
    L.omniseg_comm_init.restype = i32
    L.omniseg_segment_band.argtypes = [vp, vp, i64, i64, i64, i64, i32, i32, i32, vp, vp, i32, vp, vp, vp]
    L.omniseg_segment_band.restype = i32
    L.omniseg_gather_bands.argtypes = [vp, i32, i64, i64, i32, vp, vp, i32, vp, vp, vp, vp]
    L.omniseg_gather_bands.restype = i32
    L.omniseg_band_rows.argtypes = [i64, i64, i64, i32, i32, C.POINTER(i64), C.POINTER(i64)]
    L.omniseg_band_rows.restype = i32
    L.omniseg_render_overlay.argtypes = [vp, vp, i64, i64, vp, vp, vp, i32, vp, vp]
    L.omniseg_render_overlay.restype = i32
    L.omniseg_get_tiles.argtypes = [vp, vp, i64, C.POINTER(i64)]
    L.omniseg_get_tiles.restype = i32
    L.omniseg_get_fgmask.argtypes = [vp, vp, i64, C.POINTER(i64), C.POINTER(i64), C.POINTER(i32), C.POINTER(i32)]
    L.omniseg_get_fgmask.restype = i32
    L.omniseg_get_timings.argtypes = [vp, vp, i32]
    L.omniseg_get_timings.restype = i32
    L.omniseg_set_stream.argtypes = [vp, vp]
    L.omniseg_set_stream.restype = i32
    L.omniseg_last_error.argtypes = []
    L.omniseg_last_error.restype = C.c_char_p
    L.omniseg_destroy.argtypes = [vp]
    L.omniseg_destroy.restype = None
    L.omniseg_debug_predict_tiles.argtypes = [vp, vp, i32, i32, vp, vp, i32, vp, vp, vp]
    L.omniseg_debug_predict_tiles.restype = i32
    L.omniseg_debug_conv.argtypes = [vp, vp, i32, i32, i32, i32, vp, vp, i32, i32, i32, vp, i32, vp]
    L.omniseg_debug_conv.restype = i32
    L.omniseg_debug_set_profile.argtypes = [vp, i32]
    L.omniseg_debug_set_profile.restype = i32
    L.omniseg_debug_get_profile.argtypes = [vp, vp, i32, C.POINTER(i32)]
    L.omniseg_debug_get_profile.restype = i32
    L.omniseg_debug_band_globals.argtypes = [vp, vp, vp]
    L.omniseg_debug_band_globals.restype = i32
    L.omniseg_debug_band_fg.argtypes = [vp, vp, i64]
    L.omniseg_debug_band_fg.restype = i32
    L.omniseg_debug_get_detection.argtypes = [vp, vp, vp]
    L.omniseg_debug_get_detection.restype = i32
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        raise OmnisegError(rc, load().omniseg_last_error().decode())


def _ptr(x):
    """Raw pointer of a numpy array or torch tensor (host or device), or None."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous()
        return x.data_ptr()
    import numpy as np
    assert isinstance(x, np.ndarray) and x.flags["C_CONTIGUOUS"]
    return x.ctypes.data


def _ints(v):
    arr = (C.c_int * len(v))(*[int(x) for x in v])
    return arr


def band_rows(H, row0, row1, pad, f):
    a, b = C.c_int64(), C.c_int64()
    _check(load().omniseg_band_rows(H, row0, row1, pad, f, C.byref(a), C.byref(b)))
    return a.value, b.value


class Omniseg:
    """One predictor on one GPU (omniseg_create / omniseg_destroy)."""

    def __init__(self, arch: str, weights):
        L = load()
        import numpy as np
        if hasattr(weights, "data_ptr"):
            nbytes = weights.numel() * weights.element_size()
        else:
            weights = np.ascontiguousarray(weights, dtype="<f4")
            nbytes = weights.nbytes
        self._keep = weights
        h = L.omniseg_create(arch.encode(), _ptr(weights), nbytes)
        if not h:
            raise OmnisegError(-1, L.omniseg_last_error().decode())
        self.h = h
        self.arch = arch

    def close(self):
        if getattr(self, "h", None):
            load().omniseg_destroy(self.h)
            self.h = None

    __del__ = close

    def set_stream(self, stream_ptr):
        _check(load().omniseg_set_stream(self.h, stream_ptr))

    def output_size(self, H, W, scale):
        return load().omniseg_output_size(self.h, H, W, scale)

    def segment_slide(self, rgb, H, W, pad, patch, stride, scales, classes, out_prob=None, out_mask=None,
                      out_area=None):
        _check(load().omniseg_segment_slide(self.h, _ptr(rgb), H, W, pad, patch, stride, _ints(scales),
                                            _ints(classes), len(scales), _ptr(out_prob), _ptr(out_mask),
                                            _ptr(out_area)))

    def render_overlay(self, rgb, H, W, masks, scales, classes, out40=None, out10=None):
        """40x merge + colour overlay (+ 10x) of segment_slide masks (include/omniseg.h)."""
        _check(load().omniseg_render_overlay(self.h, _ptr(rgb), H, W, _ptr(masks), _ints(scales), _ints(classes),
                                             len(scales), _ptr(out40), _ptr(out10)))

    def comm_init(self, uid_bytes: bytes, world: int, rank: int):
        buf = C.create_string_buffer(bytes(uid_bytes), 128)
        _check(load().omniseg_comm_init(self.h, buf, world, rank))

    def segment_band(self, rgb_band, H, W, row0, row1, pad, patch, stride, scales, classes, out_prob=None,
                     out_mask=None, out_area=None):
        _check(load().omniseg_segment_band(self.h, _ptr(rgb_band), H, W, row0, row1, pad, patch, stride,
                                           _ints(scales), _ints(classes), len(scales), _ptr(out_prob),
                                           _ptr(out_mask), _ptr(out_area)))

    def gather_bands(self, root, H, W, pad, cuts, scales, band_prob=None, band_mask=None, out_prob=None,
                     out_mask=None):
        """NCCL gather of every rank's owned canvas rows into full outputs on `root` (omniseg.h)."""
        cc = (C.c_int64 * len(cuts))(*[int(c) for c in cuts])
        _check(load().omniseg_gather_bands(self.h, root, H, W, pad, cc, _ints(scales), len(scales), _ptr(band_prob),
                                           _ptr(band_mask), _ptr(out_prob), _ptr(out_mask)))

    def tiles(self):
        import numpy as np
        n = C.c_int64()
        _check(load().omniseg_get_tiles(self.h, None, 0, C.byref(n)))
        out = np.zeros(max(n.value, 1), np.uint32)
        _check(load().omniseg_get_tiles(self.h, out.ctypes.data, n.value, C.byref(n)))
        return out[:n.value]

    def fgmask(self):
        import numpy as np
        h8, w8, t, gp = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
        _check(load().omniseg_get_fgmask(self.h, None, 0, C.byref(h8), C.byref(w8), C.byref(t), C.byref(gp)))
        m = np.zeros((h8.value, w8.value), np.uint8)
        _check(load().omniseg_get_fgmask(self.h, m.ctypes.data, m.size, C.byref(h8), C.byref(w8), C.byref(t),
                                         C.byref(gp)))
        return m, t.value, gp.value

    def timings(self):
        import numpy as np
        out = np.zeros(11, np.float64)
        _check(load().omniseg_get_timings(self.h, out.ctypes.data, 11))
        return out

    def band_globals(self, pc=None, hist=None):
        import numpy as np
        if pc is None:
            _check(load().omniseg_debug_band_globals(self.h, None, None))
            return
        pc = np.ascontiguousarray(pc, np.uint8)
        hist = np.ascontiguousarray(hist, np.uint64)
        _check(load().omniseg_debug_band_globals(self.h, pc.ctypes.data, hist.ctypes.data))

    def band_fg(self, fg8=None):
        """Inject the whole slide's pre-filter level-8 foreground (band fgmin emulation)."""
        import numpy as np
        if fg8 is None:
            _check(load().omniseg_debug_band_fg(self.h, None, 0))
            return
        fg8 = np.ascontiguousarray(fg8, np.uint8)
        self._fg8 = fg8
        _check(load().omniseg_debug_band_fg(self.h, fg8.ctypes.data, fg8.size))

    def detection(self):
        import numpy as np
        pc = np.zeros(3, np.uint8)
        hist = np.zeros(256, np.uint64)
        _check(load().omniseg_debug_get_detection(self.h, pc.ctypes.data, hist.ctypes.data))
        return pc, hist

    def set_profile(self, on=True):
        _check(load().omniseg_debug_set_profile(self.h, 1 if on else 0))

    def profile(self):
        """dict(ms, flops, launches, layers=[(ms, flops, launches), ...]) of the conv launches."""
        import numpy as np
        nl = C.c_int()
        out = np.zeros(3 + 3 * 64, np.float64)
        _check(load().omniseg_debug_get_profile(self.h, out.ctypes.data, out.size, C.byref(nl)))
        layers = [tuple(out[3 + 3 * i:6 + 3 * i]) for i in range(nl.value)]
        return dict(ms=out[0], flops=out[1], launches=int(out[2]), layers=layers)

    def predict_tiles(self, tiles_u8, tasks, with_F=False, with_g=False, c_bottleneck=None):
        """tiles_u8: n x P x P x 3 uint8; tasks: list of (class, scale index)."""
        import numpy as np
        n, P = tiles_u8.shape[0], tiles_u8.shape[1]
        out_p = np.zeros((n, len(tasks), P, P), np.float32)
        out_F = np.zeros((n, P, P, 8), np.float32) if with_F else None
        out_g = np.zeros((n, c_bottleneck), np.float32) if with_g else None
        _check(load().omniseg_debug_predict_tiles(self.h, _ptr(tiles_u8), n, P, _ints([c for c, _ in tasks]),
                                                  _ints([s for _, s in tasks]), len(tasks), _ptr(out_p),
                                                  _ptr(out_g), _ptr(out_F)))
        return out_p, out_F, out_g

    def conv(self, x, w, b, stride=1, r=None, mode=0, split=False, rc=False, res_nhwc=False):
        """x: float32 [B][H][W][Cin]; w: [Cout][k][k][Cin]; returns float32 output.
        split: False (plain 16-bit storage), True / "x2" (hi + lo 16-bit), "f8" (fp16 + e4m3 lo).
        rc: residual and output in the row-chunked layout (where the width allows; the input is
        row-chunked whenever the no-swizzle multi-row kernel runs)."""
        import numpy as np
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        B, H, W, Cin = x.shape
        Cout, k = w.shape[0], w.shape[1]
        Ho, Wo = (H - 1) // stride + 1, (W - 1) // stride + 1
        if mode == 2:
            Ho, Wo = 2 * Ho, 2 * Wo
        y = np.zeros((B, Ho, Wo, Cout), np.float32)
        rr = None if r is None else np.ascontiguousarray(r, np.float32)
        _check(load().omniseg_debug_conv(self.h, _ptr(x), B, H, W, Cin, _ptr(w), _ptr(b), Cout, k, stride,
                                         _ptr(rr), mode | (32 if split == "f8" else 16 if split else 0) | (64 if rc else 0) | (128 if res_nhwc else 0),
                                         _ptr(y)))
        return y
