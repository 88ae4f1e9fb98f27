"""Thin ctypes binding of ``include/sp.h`` (argument marshalling only).

Every step of the Spatial Pooler runs in ``libsp.so``'s CUDA kernels; this
module only checks tensor shapes/dtypes/devices (the C ABI cannot check raw
pointers: SP_E_SHAPE), passes pointers and streams, and converts errors into
exceptions.  torch is used for device memory and streams only.  There is no
CPU fallback: if ``libsp.so`` is missing or has no GPU, calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SP_LIB_PATH: development A/B runs of alternative in-tree builds (scripts/_*); default libsp.so
LIB_PATH = os.environ.get("SP_LIB_PATH") or os.path.join(HERE, "libsp.so")

SP_OK, SP_E_CONFIG, SP_E_ARG, SP_E_SHAPE, SP_E_CUDA, SP_E_OOM, SP_E_STATE = range(7)
SP_PATH_AUTO, SP_PATH_PER_INPUT, SP_PATH_BATCHED = 0, 1, 2
SP_FLAG_RECORD_OVERLAPS = 1
SP_FLAG_LEARN_GRID = 2
SP_FLAG_FULL_LEARNING = 4
SP_FLAG_PATCH_GATHER = 8
SP_FLAG_PATCH_TENSOR = 16
SP_LEARN_PER_INPUT, SP_LEARN_CLUSTER, SP_LEARN_GRID = 0, 1, 2


def learn_path_name(info):
    """Human-readable learning path of the last learn=1 call (sp_info.last_learn_path)."""
    return {SP_LEARN_PER_INPUT: "per-input kernels",
            SP_LEARN_CLUSTER: f"cluster-resident kernel, {info['learn_cluster']} CTAs",
            SP_LEARN_GRID: f"grid-resident kernel, {info['learn_grid_ctas']} CTAs"}[info["last_learn_path"]]

STATUS_NAMES = {0: "SP_OK", 1: "SP_E_CONFIG", 2: "SP_E_ARG", 3: "SP_E_SHAPE", 4: "SP_E_CUDA",
                5: "SP_E_OOM", 6: "SP_E_STATE"}

# exported symbols of include/sp.h and include/sp_synth.h (checked by the CPU tests)
ABI_SYMBOLS = ("sp_config_default", "sp_create", "sp_destroy", "sp_compute", "sp_winners",
               "sp_overlaps", "sp_get_state", "sp_set_state", "sp_compute_host", "sp_plan",
               "sp_init_pools_host", "sp_get_info", "sp_last_error", "sp_version",
               "sp_get_learning_state", "sp_set_learning_state", "sp_histograms",
               "sp_compute_into", "sp_synth_frames", "sp_synth_bgr_frames", "sp_encoder_config_default",
               "sp_encoder_create", "sp_encoder_destroy", "sp_encode", "sp_encoder_get_info",
               "sp_encoder_last_error", "sp_encode_compute", "sp_pack_frames", "sp_compute_packed", "sp_compute_packed_host")


class SpError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


class SpConfig(ctypes.Structure):
    _fields_ = [
        ("input_width", ctypes.c_uint32), ("input_height", ctypes.c_uint32),
        ("patch_width", ctypes.c_uint32), ("patch_height", ctypes.c_uint32),
        ("num_columns", ctypes.c_uint32), ("synapses_per_column", ctypes.c_uint32),
        ("min_overlap", ctypes.c_uint32), ("winners_set_size", ctypes.c_uint32),
        ("inhibition_radius", ctypes.c_uint32),
        ("perm_increment", ctypes.c_float), ("perm_decrement", ctypes.c_float),
        ("initial_permanence", ctypes.c_float), ("connected_threshold", ctypes.c_float),
        ("seed", ctypes.c_uint64), ("device", ctypes.c_int32),
        ("max_inputs", ctypes.c_uint32), ("flags", ctypes.c_uint32),
        ("force_path", ctypes.c_uint32),
        ("duty_cycle_period", ctypes.c_uint32), ("max_boost", ctypes.c_float),
    ]


class SpPlanInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in (
        "path", "input_bits", "inputs_per_frame", "num_inputs", "columns_padded", "sdr_words",
        "groups", "cluster", "ctas", "window_bits", "num_windows", "chunk_bits", "stages",
        "smem_bytes", "reason", "tensor_cores", "group_inputs", "global_split")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class SpEncoderConfig(ctypes.Structure):
    _fields_ = [("src_width", ctypes.c_uint32), ("src_height", ctypes.c_uint32),
                ("dst_width", ctypes.c_uint32), ("dst_height", ctypes.c_uint32),
                ("block_size", ctypes.c_uint32), ("bias", ctypes.c_float), ("device", ctypes.c_int32)]


class SpEncoderInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("band_rows", "bands", "stages", "stage_bytes", "smem_bytes",
                                               "ctas_per_sm", "xfast")] + \
               [("kernel_launches", ctypes.c_uint64), ("kernel", ctypes.c_float * 16),
                ("chunk_frames", ctypes.c_uint32), ("l2_window_set", ctypes.c_uint32),
                ("l2_window_bytes", ctypes.c_uint64)]


class SpInfo(ctypes.Structure):
    _fields_ = [("plan", SpPlanInfo), ("kernel_launches", ctypes.c_uint64),
                ("last_num_inputs", ctypes.c_uint32), ("ell_slots", ctypes.c_uint32),
                ("sm_count", ctypes.c_int32), ("max_smem_optin", ctypes.c_int32),
                ("learn_cluster", ctypes.c_uint32), ("last_learn_cluster", ctypes.c_uint32),
                ("learn_grid_ctas", ctypes.c_uint32), ("last_learn_path", ctypes.c_uint32)]


_lib = None


def lib() -> ctypes.CDLL:
    """Loads libsp.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: run __graft_entry__.build() "
                          "(python -m paper_1608_01966_b200.build)")
    L = ctypes.CDLL(LIB_PATH)
    vp, u32, i32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int32, ctypes.c_uint64
    P = ctypes.POINTER
    sig = {
        "sp_config_default": [P(SpConfig)],
        "sp_create": [P(SpConfig), P(vp)],
        "sp_destroy": [vp],
        "sp_compute": [vp, vp, u32, ctypes.c_int, vp],
        "sp_compute_into": [vp, vp, u32, ctypes.c_int, vp, vp, vp],
        "sp_winners": [vp, vp, vp, vp],
        "sp_overlaps": [vp, vp, vp, vp],
        "sp_get_state": [vp, vp, vp, vp],
        "sp_set_state": [vp, vp, vp, vp],
        "sp_compute_host": [vp, vp, u32, ctypes.c_int, vp, vp, vp],
        "sp_pack_frames": [vp, vp, u32, vp, vp],
        "sp_compute_packed": [vp, vp, u32, vp, vp, vp],
        "sp_compute_packed_host": [vp, vp, u32, vp, vp, vp],
        "sp_plan": [P(SpConfig), u32, i32, P(SpPlanInfo)],
        "sp_init_pools_host": [P(SpConfig), vp],
        "sp_get_info": [vp, P(SpInfo)],
        "sp_get_learning_state": [vp, vp, vp, vp, vp],
        "sp_set_learning_state": [vp, vp, vp, u32],
        "sp_histograms": [vp, vp, u32, vp, vp, vp],
        "sp_synth_frames": [vp, u64, u32, u32, u32, u64, u32, u32, vp],
        "sp_synth_bgr_frames": [vp, u64, u32, u32, u32, u64, vp],
        "sp_encoder_config_default": [P(SpEncoderConfig)],
        "sp_encoder_create": [P(SpEncoderConfig), P(vp)],
        "sp_encoder_destroy": [vp],
        "sp_encode": [vp, vp, u32, vp, vp],
        "sp_encode_compute": [vp, vp, vp, u32, vp, vp, vp],
        "sp_encoder_get_info": [vp, P(SpEncoderInfo)],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.sp_last_error.restype = ctypes.c_char_p
    L.sp_last_error.argtypes = []
    L.sp_version.restype = ctypes.c_char_p
    L.sp_version.argtypes = []
    L.sp_encoder_last_error.restype = ctypes.c_char_p
    L.sp_encoder_last_error.argtypes = []
    _lib = L
    return L


def _check(status: int):
    if status != SP_OK:
        raise SpError(status, lib().sp_last_error().decode())


def make_config(**kw) -> SpConfig:
    cfg = SpConfig()
    _check(lib().sp_config_default(ctypes.byref(cfg)))
    for k, v in kw.items():
        if not hasattr(cfg, k):
            raise SpError(SP_E_CONFIG, f"unknown config key {k!r}")
        setattr(cfg, k, v)
    return cfg


def plan(num_frames: int, sm_count: int = 0, **kw) -> dict:
    out = SpPlanInfo()
    _check(lib().sp_plan(ctypes.byref(make_config(**kw)), num_frames, sm_count, ctypes.byref(out)))
    return out.as_dict()


def init_pools_host(**kw) -> np.ndarray:
    cfg = make_config(**kw)
    C, S = cfg.num_columns, cfg.synapses_per_column
    out = np.empty((C, S), dtype=np.uint32)
    _check(lib().sp_init_pools_host(ctypes.byref(cfg), out.ctypes.data))
    return out


def _stream_ptr(stream, device):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _require(t, dtype, device, shape=None, name="tensor"):
    import torch
    if not isinstance(t, torch.Tensor):
        raise SpError(SP_E_SHAPE, f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise SpError(SP_E_SHAPE, f"{name} dtype {t.dtype} != {dtype}")
    if t.device.type != "cuda" or t.device.index != device:
        raise SpError(SP_E_SHAPE, f"{name} must live on cuda:{device}, got {t.device}")
    if not t.is_contiguous():
        raise SpError(SP_E_SHAPE, f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise SpError(SP_E_SHAPE, f"{name} shape {tuple(t.shape)} != {tuple(shape)}")


def _host_buffer(a, dtype, shape, name):
    """Checks a host buffer (numpy array or CPU torch tensor) for a host-pointer entry point and
    returns its address: the C ABI copies exactly the bytes the shape implies, so a short,
    mistyped or strided buffer would be overrun silently (heap corruption) without this check."""
    import torch
    if isinstance(a, torch.Tensor):
        if a.device.type != "cpu":
            raise SpError(SP_E_SHAPE, f"{name} must be a host (CPU) buffer, got {a.device}")
        tdt = {np.uint8: torch.uint8, np.uint32: (torch.uint32, torch.int32)}[dtype]
        ok = a.dtype in tdt if isinstance(tdt, tuple) else a.dtype == tdt
        if not ok:
            raise SpError(SP_E_SHAPE, f"{name} dtype {a.dtype} is not {np.dtype(dtype).name}")
        if not a.is_contiguous():
            raise SpError(SP_E_SHAPE, f"{name} must be C-contiguous")
        got, addr = tuple(a.shape), a.data_ptr()
    elif isinstance(a, np.ndarray):
        ok = a.dtype == dtype or (dtype is np.uint32 and a.dtype == np.int32)
        if not ok:
            raise SpError(SP_E_SHAPE, f"{name} dtype {a.dtype} is not {np.dtype(dtype).name}")
        if not a.flags["C_CONTIGUOUS"]:
            raise SpError(SP_E_SHAPE, f"{name} must be C-contiguous")
        if name != "frames" and name != "planes" and not a.flags["WRITEABLE"]:
            raise SpError(SP_E_SHAPE, f"{name} must be writeable")
        got, addr = tuple(a.shape), a.ctypes.data
    else:
        raise SpError(SP_E_SHAPE, f"{name} must be a numpy array or a CPU torch.Tensor")
    if got != tuple(shape):
        raise SpError(SP_E_SHAPE, f"{name} shape {got} != {tuple(shape)}")
    return addr


def synth_frames(out, first_frame: int, seed: int, rho: float = 0.5, nonzero: str = "255",
                 stream=None):
    """Fills uint8 cuda tensor ``out[F, H, W]`` with frames of the seeded stream (bench/test)."""
    import torch
    _require(out, torch.uint8, out.device.index if out.is_cuda else -1, name="out")
    F, H, W = out.shape
    mode = {"255": 0, "1": 1, "random": 2}[nonzero]
    q24 = int(round(rho * (1 << 24)))
    _check(lib().sp_synth_frames(ctypes.c_void_p(out.data_ptr()), first_frame, F, H, W, seed, q24,
                                 mode, _stream_ptr(stream, out.device)))
    return out


def synth_bgr_frames(out, first_frame: int, seed: int, stream=None):
    """Fills uint8 cuda tensor ``out[F, H, W, 3]`` with BGR frames of the seeded recipe (bench/test)."""
    import torch
    _require(out, torch.uint8, out.device.index if out.is_cuda else -1, name="out")
    F, H, W, ch = out.shape
    if ch != 3:
        raise SpError(SP_E_SHAPE, "out must be [F, H, W, 3]")
    _check(lib().sp_synth_bgr_frames(ctypes.c_void_p(out.data_ptr()), first_frame, F, H, W, seed,
                                     _stream_ptr(stream, out.device)))
    return out


class Encoder:
    """The on-device adaptive video encoder (``include/sp_encoder.h``, NEXT-3): BGR frames ->
    binarised frames for ``SpatialPooler.compute``."""

    def __init__(self, **kw):
        cfg = SpEncoderConfig()
        _check(lib().sp_encoder_config_default(ctypes.byref(cfg)))
        for k, v in kw.items():
            if not hasattr(cfg, k):
                raise SpError(SP_E_CONFIG, f"unknown encoder config key {k!r}")
            setattr(cfg, k, v)
        self.cfg = cfg
        h = ctypes.c_void_p()
        st = lib().sp_encoder_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != SP_OK:
            raise SpError(st, lib().sp_encoder_last_error().decode())
        self._h = h
        self.device = int(cfg.device)
        self.src_shape = (int(cfg.src_height), int(cfg.src_width), 3)
        self.dst_shape = (int(cfg.dst_height), int(cfg.dst_width))

    def close(self):
        if getattr(self, "_h", None):
            lib().sp_encoder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def encode(self, bgr, out=None, stream=None):
        """``bgr``: uint8 cuda [F, H0, W0, 3] -> uint8 cuda [F, H1, W1] (255 / 0)."""
        import torch
        _require(bgr, torch.uint8, self.device, name="bgr")
        if bgr.dim() != 4 or tuple(bgr.shape[1:]) != self.src_shape:
            raise SpError(SP_E_SHAPE, f"bgr must be [F, {self.src_shape}]")
        F = bgr.shape[0]
        if out is None:
            out = torch.empty((F, *self.dst_shape), dtype=torch.uint8, device=bgr.device)
        _require(out, torch.uint8, self.device, (F, *self.dst_shape), "out")
        st = lib().sp_encode(self._h, ctypes.c_void_p(bgr.data_ptr()), F, ctypes.c_void_p(out.data_ptr()),
                             _stream_ptr(stream, bgr.device))
        if st != SP_OK:
            raise SpError(st, lib().sp_encoder_last_error().decode())
        return out

    def encode_compute(self, sp, bgr, sdr=None, counts=None, stream=None):
        """Raw BGR video -> SDRs in one call (``sp_encode_compute``): ``bgr`` uint8 cuda
        [F, H0, W0, 3] through the encoder and ``sp``'s inference, the binarised frames held in
        a persisting-L2 chunk buffer between the two.  Returns (sdr int32 [F*P, words],
        counts int32 [F*P])."""
        import torch
        _require(bgr, torch.uint8, self.device, name="bgr")
        if bgr.dim() != 4 or tuple(bgr.shape[1:]) != self.src_shape:
            raise SpError(SP_E_SHAPE, f"bgr must be [F, {self.src_shape}]")
        n = bgr.shape[0] * sp.inputs_per_frame
        if sdr is None:
            sdr = torch.empty((n, sp.sdr_words), dtype=torch.int32, device=bgr.device)
        if counts is None:
            counts = torch.empty((n,), dtype=torch.int32, device=bgr.device)
        _require(sdr, torch.int32, self.device, (n, sp.sdr_words), "sdr")
        _require(counts, torch.int32, self.device, (n,), "counts")
        st = lib().sp_encode_compute(self._h, sp._h, ctypes.c_void_p(bgr.data_ptr()), bgr.shape[0],
                                     ctypes.c_void_p(sdr.data_ptr()), ctypes.c_void_p(counts.data_ptr()),
                                     _stream_ptr(stream, bgr.device))
        if st != SP_OK:
            raise SpError(st, lib().sp_encoder_last_error().decode())
        sp.last_num_inputs = n
        return sdr, counts

    def info(self) -> dict:
        out = SpEncoderInfo()
        _check(lib().sp_encoder_get_info(self._h, ctypes.byref(out)))
        d = {n: int(getattr(out, n)) for n, _ in out._fields_ if n != "kernel"}
        d["kernel"] = list(out.kernel)[:int(self.cfg.block_size)]
        return d


class SpatialPooler:
    """One SP instance (a ``sp_handle``) on one CUDA device."""

    def __init__(self, **kw):
        self.cfg = make_config(**kw)
        h = ctypes.c_void_p()
        _check(lib().sp_create(ctypes.byref(self.cfg), ctypes.byref(h)))
        self._h = h
        self.device = int(self.cfg.device)
        self.C = int(self.cfg.num_columns)
        self.S = int(self.cfg.synapses_per_column)
        W, H = int(self.cfg.input_width), int(self.cfg.input_height)
        pw = int(self.cfg.patch_width) or W
        ph = int(self.cfg.patch_height) or H
        self.frame_shape = (H, W)
        self.inputs_per_frame = (W // pw) * (H // ph)
        self.sdr_words = (self.C + 31) // 32
        # bit-plane input: words per frame = ceil(W*H/32) rounded up to 4
        self.packed_words = ((H * W + 31) // 32 + 3) // 4 * 4
        self.last_num_inputs = 0

    # -- lifetime ---------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().sp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- hot path ---------------------------------------------------------------------
    def compute(self, frames, learn: bool = False, stream=None) -> int:
        """``frames``: uint8 cuda tensor [F, H, W]. Returns the number of SP inputs."""
        import torch
        _require(frames, torch.uint8, self.device, name="frames")
        if frames.dim() != 3 or tuple(frames.shape[1:]) != self.frame_shape:
            raise SpError(SP_E_SHAPE, f"frames must be [F, {self.frame_shape[0]}, {self.frame_shape[1]}]")
        F = frames.shape[0]
        _check(lib().sp_compute(self._h, ctypes.c_void_p(frames.data_ptr()), F, int(bool(learn)),
                                _stream_ptr(stream, frames.device)))
        self.last_num_inputs = F * self.inputs_per_frame
        self._res = None
        return self.last_num_inputs

    def compute_into(self, frames, sdr, counts, learn: bool = False, stream=None) -> int:
        """``compute`` with the winners written straight into ``sdr`` (int32 [n, words]) and
        ``counts`` (int32 [n]) cuda tensors (no copy afterwards)."""
        import torch
        _require(frames, torch.uint8, self.device, name="frames")
        if frames.dim() != 3 or tuple(frames.shape[1:]) != self.frame_shape:
            raise SpError(SP_E_SHAPE, f"frames must be [F, {self.frame_shape[0]}, {self.frame_shape[1]}]")
        n = frames.shape[0] * self.inputs_per_frame
        _require(sdr, torch.int32, self.device, (n, self.sdr_words), "sdr")
        _require(counts, torch.int32, self.device, (n,), "counts")
        _check(lib().sp_compute_into(self._h, ctypes.c_void_p(frames.data_ptr()), frames.shape[0],
                                     int(bool(learn)), ctypes.c_void_p(sdr.data_ptr()),
                                     ctypes.c_void_p(counts.data_ptr()), _stream_ptr(stream, frames.device)))
        self.last_num_inputs = n
        self._res = (sdr, counts)  # keep the result buffers alive until the next call
        return n

    # -- bit-plane input (include/sp.h "bit-plane input") ---------------------------
    def pack_frames(self, frames, planes=None, stream=None):
        """uint8 cuda frames [F, H, W] -> int32-view bit-planes [F, packed_words] (sp_pack_frames)."""
        import torch
        _require(frames, torch.uint8, self.device, name="frames")
        if frames.dim() != 3 or tuple(frames.shape[1:]) != self.frame_shape:
            raise SpError(SP_E_SHAPE, f"frames must be [F, {self.frame_shape[0]}, {self.frame_shape[1]}]")
        F = frames.shape[0]
        if planes is None:
            planes = torch.empty((F, self.packed_words), dtype=torch.int32, device=frames.device)
        _require(planes, torch.int32, self.device, (F, self.packed_words), "planes")
        _check(lib().sp_pack_frames(self._h, ctypes.c_void_p(frames.data_ptr()), F,
                                    ctypes.c_void_p(planes.data_ptr()), _stream_ptr(stream, frames.device)))
        return planes

    def compute_packed(self, planes, sdr=None, counts=None, stream=None) -> int:
        """Inference on bit-planes (int32-view uint32 [F, packed_words] cuda tensor); winners into
        ``sdr`` / ``counts`` when given, else kept for ``winners()``."""
        import torch
        _require(planes, torch.int32, self.device, name="planes")
        if planes.dim() != 2 or planes.shape[1] != self.packed_words:
            raise SpError(SP_E_SHAPE, f"planes must be [F, {self.packed_words}]")
        n = planes.shape[0] * self.inputs_per_frame
        if (sdr is None) != (counts is None):
            raise SpError(SP_E_ARG, "give both sdr and counts, or neither")
        if sdr is not None:
            _require(sdr, torch.int32, self.device, (n, self.sdr_words), "sdr")
            _require(counts, torch.int32, self.device, (n,), "counts")
        _check(lib().sp_compute_packed(self._h, ctypes.c_void_p(planes.data_ptr()), planes.shape[0],
                                       ctypes.c_void_p(sdr.data_ptr()) if sdr is not None else None,
                                       ctypes.c_void_p(counts.data_ptr()) if counts is not None else None,
                                       _stream_ptr(stream, planes.device)))
        self.last_num_inputs = n
        self._res = (sdr, counts) if sdr is not None else None
        return n

    def compute_packed_host_into(self, planes, sdr, counts, stream=None):
        """End-to-end bit-plane inference with host buffers (numpy arrays or pinned torch CPU
        tensors): planes uint32 [F, packed_words] -> sdr uint32 [n, words], counts uint32 [n]
        (or None).  Shapes, dtypes and contiguity are checked here (SP_E_SHAPE)."""
        import torch
        if getattr(planes, "ndim", 0) != 2:
            raise SpError(SP_E_SHAPE, f"planes must be [F, {self.packed_words}]")
        F = int(planes.shape[0])
        n = F * self.inputs_per_frame
        pp = _host_buffer(planes, np.uint32, (F, self.packed_words), "planes")
        sp_ = _host_buffer(sdr, np.uint32, (n, self.sdr_words), "sdr")
        cp = _host_buffer(counts, np.uint32, (n,), "counts") if counts is not None else None
        _check(lib().sp_compute_packed_host(self._h, ctypes.c_void_p(pp), F, ctypes.c_void_p(sp_),
                                            ctypes.c_void_p(cp) if cp is not None else None,
                                            _stream_ptr(stream, torch.device("cuda", self.device))))
        self.last_num_inputs = n

    def winners(self, sdr=None, counts=None, stream=None):
        """SDRs of the last call: (uint32 [n, words] as int32 view, int32 [n]) cuda tensors."""
        import torch
        n = self.last_num_inputs
        dev = torch.device("cuda", self.device)
        if sdr is None:
            sdr = torch.empty((n, self.sdr_words), dtype=torch.int32, device=dev)
        if counts is None:
            counts = torch.empty((n,), dtype=torch.int32, device=dev)
        _require(sdr, torch.int32, self.device, (n, self.sdr_words), "sdr")
        _require(counts, torch.int32, self.device, (n,), "counts")
        _check(lib().sp_winners(self._h, ctypes.c_void_p(sdr.data_ptr()),
                                ctypes.c_void_p(counts.data_ptr()), _stream_ptr(stream, dev)))
        return sdr, counts

    def overlaps(self, stream=None):
        """(raw uint16-as-int16 [n, C], boosted float32 [n, C]) of the last call."""
        import torch
        n = self.last_num_inputs
        dev = torch.device("cuda", self.device)
        raw = torch.empty((n, self.C), dtype=torch.int16, device=dev)
        boosted = torch.empty((n, self.C), dtype=torch.float32, device=dev)
        _check(lib().sp_overlaps(self._h, ctypes.c_void_p(raw.data_ptr()),
                                 ctypes.c_void_p(boosted.data_ptr()), _stream_ptr(stream, dev)))
        return raw, boosted

    def histograms(self, video_offsets, counts=None, hist=None, stream=None):
        """Per-video SDR histograms of the last call (NEXT-4): video v = SP inputs
        [offsets[v], offsets[v+1]).  Returns (counts int32-view uint32 [V, C], hist f32 [V, C])."""
        import torch
        off = np.ascontiguousarray(video_offsets, dtype=np.uint32)
        V = len(off) - 1
        dev = torch.device("cuda", self.device)
        if counts is None:
            counts = torch.empty((V, self.C), dtype=torch.int32, device=dev)
        if hist is None:
            hist = torch.empty((V, self.C), dtype=torch.float32, device=dev)
        _require(counts, torch.int32, self.device, (V, self.C), "counts")
        _require(hist, torch.float32, self.device, (V, self.C), "hist")
        _check(lib().sp_histograms(self._h, ctypes.c_void_p(off.ctypes.data), V,
                                   ctypes.c_void_p(counts.data_ptr()), ctypes.c_void_p(hist.data_ptr()),
                                   _stream_ptr(stream, dev)))
        return counts, hist

    def compute_host(self, frames: np.ndarray, learn: bool = False, stream=None):
        """End-to-end call with host buffers (H2D/D2H inside): returns (sdr uint32, counts uint32)."""
        frames = np.ascontiguousarray(frames, dtype=np.uint8)
        if frames.ndim != 3 or frames.shape[1:] != self.frame_shape:
            raise SpError(SP_E_SHAPE, "frames must be [F, H, W] uint8")
        n = frames.shape[0] * self.inputs_per_frame
        sdr = np.empty((n, self.sdr_words), dtype=np.uint32)
        counts = np.empty((n,), dtype=np.uint32)
        self.compute_host_into(frames, sdr, counts, learn, stream)
        return sdr, counts

    def compute_host_into(self, frames, sdr, counts, learn: bool = False, stream=None):
        """Same with caller buffers (numpy arrays or pinned torch CPU tensors): frames uint8
        [F, H, W] -> sdr uint32 [n, words], counts uint32 [n] (or None).  Shapes, dtypes and
        contiguity are checked here (SP_E_SHAPE): the C ABI copies by the implied sizes."""
        import torch
        if getattr(frames, "ndim", 0) != 3:
            raise SpError(SP_E_SHAPE, "frames must be [F, H, W] uint8")
        F = int(frames.shape[0])
        n = F * self.inputs_per_frame
        fp = _host_buffer(frames, np.uint8, (F, *self.frame_shape), "frames")
        sp_ = _host_buffer(sdr, np.uint32, (n, self.sdr_words), "sdr")
        cp = _host_buffer(counts, np.uint32, (n,), "counts") if counts is not None else None
        _check(lib().sp_compute_host(self._h, ctypes.c_void_p(fp), F, int(bool(learn)),
                                     ctypes.c_void_p(sp_),
                                     ctypes.c_void_p(cp) if cp is not None else None,
                                     _stream_ptr(stream, torch.device("cuda", self.device))))
        self.last_num_inputs = n

    # -- state ------------------------------------------------------------------------
    def get_state(self):
        idx = np.empty((self.C, self.S), np.uint32)
        perm = np.empty((self.C, self.S), np.float32)
        boost = np.empty((self.C,), np.float32)
        _check(lib().sp_get_state(self._h, idx.ctypes.data, perm.ctypes.data, boost.ctypes.data))
        return idx, perm, boost

    def set_state(self, idx=None, perm=None, boost=None):
        def arr(a, dt, shape):
            if a is None:
                return None, None
            a = np.ascontiguousarray(a, dtype=dt)
            if a.shape != shape:
                raise SpError(SP_E_SHAPE, f"state array shape {a.shape} != {shape}")
            return a, ctypes.c_void_p(a.ctypes.data)
        i, ip = arr(idx, np.uint32, (self.C, self.S))
        p, pp = arr(perm, np.float32, (self.C, self.S))
        b, bp = arr(boost, np.float32, (self.C,))
        _check(lib().sp_set_state(self._h, ip, pp, bp))

    def get_learning_state(self):
        """Full-learning state: (active_duty f32[C], overlap_duty f32[C], radius, iteration)."""
        adc = np.empty((self.C,), np.float32)
        odc = np.empty((self.C,), np.float32)
        r = ctypes.c_uint32()
        it = ctypes.c_uint64()
        _check(lib().sp_get_learning_state(self._h, adc.ctypes.data, odc.ctypes.data,
                                           ctypes.byref(r), ctypes.byref(it)))
        return adc, odc, int(r.value), int(it.value)

    def set_learning_state(self, active_duty=None, overlap_duty=None, radius=None):
        def arr(a):
            if a is None:
                return None, None
            a = np.ascontiguousarray(a, dtype=np.float32)
            if a.shape != (self.C,):
                raise SpError(SP_E_SHAPE, f"duty array shape {a.shape} != {(self.C,)}")
            return a, ctypes.c_void_p(a.ctypes.data)
        a, ap = arr(active_duty)
        o, op = arr(overlap_duty)
        if radius is None:
            radius = self.get_learning_state()[2]
        _check(lib().sp_set_learning_state(self._h, ap, op, int(radius)))

    def info(self) -> dict:
        out = SpInfo()
        _check(lib().sp_get_info(self._h, ctypes.byref(out)))
        d = {n: (out.plan.as_dict() if n == "plan" else int(getattr(out, n))) for n, _ in out._fields_}
        return d

    def kernel_launches(self) -> int:
        return self.info()["kernel_launches"]
