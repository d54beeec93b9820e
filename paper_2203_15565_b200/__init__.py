"""B200-native Partial FC hot path — Python host mirror of the reference API.

The product is ``libpfc_gpu.so`` (hand-written sm_100a CUDA + C ABI, include/pfc_gpu.h).  This
module binds that ABI with ctypes and mirrors the reference's C++ interface for the path
(/root/reference/proj/include/pfc/):

  reference (C++)                                   here
  ------------------------------------------------  ------------------------------------------
  ShardLayout (sampler.hpp:16-33)                   ShardLayout
  buffer_capacity (sampler.hpp:50-57)               buffer_capacity
  MarginConfig::{plain,cosface_style,arcface_style} MarginConfig.{plain,cosface_style,arcface_style}
  StepConfig / StepResult (shardsim.hpp:117-135)    StepConfig / StepResult
  SeededRng / make_stream (rng.hpp:40-96)           SeededRng / make_stream
  std::vector<CenterShard> + init_center_shards     CenterShards (device-resident shards)
  distributed_partial_step (shardsim.hpp:166-420)   distributed_partial_step
  pfc::*Error (error.hpp:9-42)                      ShapeError, ContractError, CapacityError, ...

There is no CPU fallback: importing works without a GPU (so the ABI can be inspected), but
creating CenterShards needs the built library and an sm_100 device and fails loudly otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpfc_gpu.so")
ROOT = os.path.dirname(HERE)
HEADER = os.path.join(ROOT, "include", "pfc_gpu.h")

_MASK = (1 << 64) - 1
_PHI = 0x9E3779B97F4A7C15


# ----------------------------------------------------------------------------- errors
class Error(RuntimeError):
    """pfc::Error (error.hpp:9-11)."""


class ShapeError(Error):
    pass


class ContractError(Error):
    pass


class CapacityError(Error):
    pass


class ConfigError(Error):
    pass


class NumericalError(Error):
    pass


class DataError(Error):
    """error.hpp DataError (checkpoint streams, io.hpp)"""


class CudaError(Error):
    pass


class NcclError(Error):
    pass


_ERRORS = {1: ShapeError, 2: ContractError, 3: CapacityError, 4: ConfigError, 5: NumericalError,
           6: CudaError, 7: NcclError, 8: DataError}


# ----------------------------------------------------------------------------- rng.hpp mirror
def mix64(x: int) -> int:
    x &= _MASK
    x ^= x >> 33
    x = (x * 0xFF51AFD7ED558CCD) & _MASK
    x ^= x >> 33
    x = (x * 0xC4CEB9FE1A85EC53) & _MASK
    x ^= x >> 33
    return x


def fnv1a(s: str, h: int = 0xCBF29CE484222325) -> int:
    for ch in s.encode():
        h ^= ch
        h = (h * 0x100000001B3) & _MASK
    return h


def make_stream(tag: str, a: int = 0, b: int = 0) -> int:
    """rng.hpp:91-96"""
    h = fnv1a(tag)
    h = mix64(h ^ mix64((a + _PHI) & _MASK))
    h = mix64(h ^ mix64((b + 0x2545F4914F6CDD1D) & _MASK))
    return h


@dataclass(frozen=True)
class SeededRng:
    """Key of a counter-based stream (rng.hpp:40-87); the GPU sampler consumes (seed, stream)."""
    seed: int
    stream_id: int

    def fork(self, label: int) -> "SeededRng":
        return SeededRng(self.seed, mix64(self.stream_id ^ mix64((label + _PHI) & _MASK)))


# ----------------------------------------------------------------------------- config types
PLAIN, ADDITIVE_COSINE, ADDITIVE_ANGULAR = 0, 1, 2
COMBINED = 3  # extension (PFC_MARGIN_COMBINED): not a reference MarginKind


@dataclass(frozen=True)
class MarginConfig:
    """margin.hpp:17-37.  COMBINED (an extension beyond the reference) adds m1 and m3:
    s (cos(m1 theta + margin) - m3) on the positive entry; m1 / m3 are ignored otherwise."""
    kind: int = ADDITIVE_COSINE
    scale: float = 64.0
    margin: float = 0.4
    m1: float = 1.0
    m3: float = 0.0

    @staticmethod
    def plain() -> "MarginConfig":
        return MarginConfig(PLAIN, 1.0, 0.0)

    @staticmethod
    def cosface_style(s: float = 64.0, m: float = 0.4) -> "MarginConfig":
        return MarginConfig(ADDITIVE_COSINE, s, m)

    @staticmethod
    def arcface_style(s: float = 64.0, m: float = 0.5) -> "MarginConfig":
        return MarginConfig(ADDITIVE_ANGULAR, s, m)

    @staticmethod
    def combined(s: float = 64.0, m1: float = 1.0, m2: float = 0.3,
                 m3: float = 0.2) -> "MarginConfig":
        """The combined (m1, m2, m3) margin; (1, m, 0) is ArcFace, (1, 0, m) CosFace up to the
        ArcFace clamp of the cosine."""
        return MarginConfig(COMBINED, s, m2, m1, m3)

    def validate(self) -> None:
        if not self.scale > 0.0:
            raise ConfigError("margin: scale must be positive")
        if self.margin < 0.0 or self.margin >= 1.0:
            raise ConfigError("margin: m must be in [0, 1)")
        if self.kind == PLAIN and (self.scale != 1.0 or self.margin != 0.0):
            raise ConfigError("margin: plain kind requires s=1, m=0")
        if self.kind == COMBINED and not 0.0 < self.m1 <= 2.0:
            raise ConfigError("margin: m1 must be in (0, 2]")
        if self.kind == COMBINED and not 0.0 <= self.m3 < 1.0:
            raise ConfigError("margin: m3 must be in [0, 1)")


@dataclass
class StepConfig:
    """shardsim.hpp:117-127.  ``conflict`` (ConflictInfo) is used when with_diagnostics."""
    r: float = 0.1
    margin: MarginConfig = field(default_factory=MarginConfig.cosface_style)
    filter_threshold: float | None = None
    lr: float = 0.1
    momentum: float = 0.9
    weight_decay: float = 5e-4
    with_diagnostics: bool = False
    step_index: int = -1
    conflict: "ConflictInfo | None" = None


@dataclass
class ConflictInfo:
    """types.hpp:80-86: true identity of every class [C] and of every batch sample [B]."""
    class_identity: np.ndarray
    sample_identity: np.ndarray


@dataclass
class DiagnosticsSnapshot:
    """types.hpp:72-78 (metrics.hpp:56-146 as the step reports them)."""
    iteration: int = 0
    apcs: float = 0.0
    amncs: float = 0.0
    amncs_conflicted: float | None = None
    amncs_hard: float | None = None


class DiagOut(C.Structure):
    _fields_ = [("apcs", C.c_double), ("amncs", C.c_double), ("amncs_conflicted", C.c_double),
                ("amncs_hard", C.c_double), ("has_conflicted", C.c_int32),
                ("has_split", C.c_int32), ("reserved", C.c_int32 * 2)]


@dataclass
class CollectiveTrace:
    """types.hpp:51-69 (reference closed form)."""
    allgather_bytes: int = 0
    reduce_scalar_bytes: int = 0
    reduce_grad_bytes: int = 0
    reduce_ops: int = 0


@dataclass
class SampleBuffer:
    """sampler.hpp:38-46"""
    shard_id: int
    class_indices: np.ndarray
    num_positives: int


@dataclass
class StepResult:
    """shardsim.hpp:129-135"""
    loss: float
    d_features: np.ndarray | None
    trace: CollectiveTrace
    buffers: list
    diagnostics: DiagnosticsSnapshot | None = None
    # not in the reference's StepResult: what the GPU path moved (pfc_gpu_step_out)
    nccl_bytes: int = 0
    wire_bytes: int = 0


class ShardLayout:
    """sampler.hpp:16-33"""

    def __init__(self, classes: int, shards: int):
        if classes < 1 or shards < 1:
            raise ContractError("ShardLayout: need at least one class and one shard")
        self.num_classes, self.num_shards = classes, shards

    def block(self) -> int:
        return (self.num_classes + self.num_shards - 1) // self.num_shards

    def owner(self, cls: int) -> int:
        return cls // self.block()

    def owned_begin(self, k: int) -> int:
        return min(k * self.block(), self.num_classes)

    def owned_end(self, k: int) -> int:
        return min((k + 1) * self.block(), self.num_classes)

    def owned_count(self, k: int) -> int:
        return self.owned_end(k) - self.owned_begin(k)


def buffer_capacity(layout: ShardLayout, r: float) -> int:
    """sampler.hpp:50-57"""
    if not (0.0 < r <= 1.0):
        raise ContractError("buffer_capacity: sampling ratio must lie in (0, 1]")
    import math
    total = int(math.ceil(layout.num_classes * r - 1e-9))
    return (total + layout.num_shards - 1) // layout.num_shards


# ----------------------------------------------------------------------------- C ABI
class Desc(C.Structure):
    _fields_ = [("num_classes", C.c_int64), ("dim", C.c_int64), ("num_shards", C.c_int64),
                ("max_batch", C.c_int64), ("r", C.c_double), ("margin_kind", C.c_int32),
                ("margin_scale", C.c_double), ("margin_m", C.c_double),
                ("has_filter", C.c_int32), ("filter_threshold", C.c_double),
                ("momentum", C.c_double), ("weight_decay", C.c_double),
                ("precision", C.c_int32), ("device", C.c_int32), ("rank", C.c_int32),
                ("world_size", C.c_int32), ("nccl_id", C.c_void_p), ("flags", C.c_int32),
                ("margin_m1", C.c_double), ("margin_m3", C.c_double)]


class StepConfigC(C.Structure):
    _fields_ = [("r", C.c_double), ("margin_kind", C.c_int32), ("margin_scale", C.c_double),
                ("margin_m", C.c_double), ("has_filter", C.c_int32),
                ("filter_threshold", C.c_double), ("momentum", C.c_double),
                ("weight_decay", C.c_double), ("margin_m1", C.c_double),
                ("margin_m3", C.c_double)]


class StepArgs(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("stream_id", C.c_uint64), ("lr", C.c_double),
                ("step_index", C.c_int64)]


class StepOut(C.Structure):
    _fields_ = [("loss", C.c_double), ("allgather_bytes", C.c_uint64),
                ("reduce_scalar_bytes", C.c_uint64), ("reduce_grad_bytes", C.c_uint64),
                ("reduce_ops", C.c_uint64), ("capacity", C.c_int64),
                ("rejection_shards", C.c_int32), ("reserved", C.c_int32),
                ("nccl_bytes", C.c_uint64), ("wire_bytes", C.c_uint64)]


PRECISION_BF16, PRECISION_FP32, PRECISION_TF32 = 0, 1, 2
FLAG_FORCE_SEQUENTIAL_SAMPLER, FLAG_NO_GRAPH, FLAG_EXACT_SOFTMAX, FLAG_DEBUG_LOGITS = 1, 2, 4, 8
FLAG_GUARD, FLAG_NO_PDL, FLAG_WIDE_SAMPLER_CHUNKS, FLAG_FORCE_COLLECTIVES = 16, 32, 64, 128

_lib = None


def header_functions() -> list[str]:
    """Entry points declared in include/pfc_gpu.h."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pfc_gpu_\w+)\s*\(", txt)))


def load_library(path: str | None = None) -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run __graft_entry__.build() (no CPU fallback)")
    lib = C.CDLL(path)
    vp, i64, u8p = C.c_void_p, C.c_int64, C.POINTER(C.c_uint8)
    sig = {
        "pfc_gpu_create": (C.c_int, [C.POINTER(Desc), C.POINTER(vp)]),
        "pfc_gpu_destroy": (C.c_int, [vp]),
        "pfc_gpu_last_error": (C.c_char_p, [vp]),
        "pfc_gpu_nccl_unique_id": (C.c_int, [u8p]),
        "pfc_gpu_loopback_id": (C.c_int, [u8p]),
        "pfc_gpu_debug_logits": (C.c_int, [vp, vp]),
        "pfc_gpu_version": (C.c_char_p, []),
        "pfc_gpu_capacity": (i64, [vp]),
        "pfc_gpu_local_shards": (C.c_int, [vp, C.POINTER(i64), C.POINTER(i64)]),
        "pfc_gpu_shard_range": (C.c_int, [vp, i64, C.POINTER(i64), C.POINTER(i64)]),
        "pfc_gpu_set_shard": (C.c_int, [vp, i64, vp, vp]),
        "pfc_gpu_get_shard": (C.c_int, [vp, i64, vp, vp]),
        "pfc_gpu_init_shards": (C.c_int, [vp, C.c_uint64]),
        "pfc_gpu_device_state": (C.c_int, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64)]),
        "pfc_gpu_step": (C.c_int, [vp, vp, vp, i64, C.POINTER(StepArgs), vp, C.POINTER(StepOut)]),
        "pfc_gpu_step_features": (C.c_int, [vp, vp, vp, i64, C.POINTER(StepArgs), vp,
                                            C.POINTER(StepOut)]),
        "pfc_gpu_step_device": (C.c_int, [vp, vp, vp, i64, C.POINTER(StepArgs), vp,
                                          C.POINTER(StepOut)]),
        "pfc_gpu_sync": (C.c_int, [vp, C.POINTER(StepOut)]),
        "pfc_gpu_get_buffers": (C.c_int, [vp, i64, vp, C.POINTER(i64)]),
        "pfc_gpu_stream": (vp, [vp]),
        "pfc_gpu_bench_inputs": (C.c_int, [vp, C.c_uint64, C.c_uint64, i64, vp, vp]),
        "pfc_gpu_phase_times": (C.c_int, [vp, C.POINTER(C.c_float), C.POINTER(C.c_char_p),
                                          C.c_int]),
        "pfc_gpu_set_phase_timing": (C.c_int, [vp, C.c_int]),
        "pfc_gpu_launches_per_step": (i64, [vp]),
        "pfc_gpu_diagnostics": (C.c_int, [vp, vp, vp, i64, vp, vp, C.POINTER(DiagOut)]),
        "pfc_gpu_write_shards": (C.c_int, [vp, C.c_char_p, C.c_int]),
        "pfc_gpu_mics": (C.c_int, [vp, vp]),
        "pfc_gpu_read_shards": (C.c_int, [vp, C.c_char_p, i64, C.POINTER(i64)]),
        "pfc_gpu_check_guards": (C.c_int, [vp, C.POINTER(i64)]),
        "pfc_gpu_set_step_config": (C.c_int, [vp, C.POINTER(StepConfigC)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


def _check(rc: int, ctx=None) -> None:
    if rc != 0:
        msg = _lib.pfc_gpu_last_error(ctx).decode()
        raise _ERRORS.get(rc, Error)(msg)


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = (C.c_uint8 * 128)()
    _check(lib.pfc_gpu_nccl_unique_id(buf))
    return bytes(buf)


def loopback_id() -> bytes:
    """Id of a loopback communicator: world_size CenterShards created in this process (one thread
    each, e.g. all on cuda:0) act as the ranks of one job (pfc_gpu_loopback_id)."""
    lib = load_library()
    buf = (C.c_uint8 * 128)()
    _check(lib.pfc_gpu_loopback_id(buf))
    return bytes(buf)


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


class CenterShards:
    """Device-resident replacement of ``std::vector<CenterShard>`` for one rank.

    Owns W and momentum of the reference shards [rank*K/world, (rank+1)*K/world) as fp32
    row-major [classes x D] on this rank's GPU.  Every step takes its own StepConfig, like the
    reference; a changed r / margin / filter / momentum / weight decay is applied before the step
    (set_step_config), lr and the iteration rng ride with the step.
    """

    def __init__(self, layout: ShardLayout, dim: int, cfg: StepConfig, *, max_batch: int = 1024,
                 precision: int = PRECISION_BF16, device: int = 0, rank: int = 0,
                 world_size: int = 1, nccl_id: bytes | None = None, flags: int = 0):
        cfg.margin.validate()
        lib = load_library()
        self.layout, self.dim, self.cfg, self.precision = layout, dim, cfg, precision
        self.world_size, self.rank = world_size, rank
        self._nccl_id = (C.c_uint8 * 128)(*nccl_id) if nccl_id else None
        d = Desc(layout.num_classes, dim, layout.num_shards, max_batch, cfg.r, cfg.margin.kind,
                 cfg.margin.scale, cfg.margin.margin, 0 if cfg.filter_threshold is None else 1,
                 0.0 if cfg.filter_threshold is None else cfg.filter_threshold, cfg.momentum,
                 cfg.weight_decay, precision, device, rank, world_size,
                 C.cast(self._nccl_id, C.c_void_p) if self._nccl_id else None, flags,
                 cfg.margin.m1, cfg.margin.m3)
        h = C.c_void_p()
        _check(lib.pfc_gpu_create(C.byref(d), C.byref(h)), None)
        self._h = h
        self.capacity = lib.pfc_gpu_capacity(h)
        f, n = C.c_int64(), C.c_int64()
        lib.pfc_gpu_local_shards(h, C.byref(f), C.byref(n))
        self.local_shards = list(range(f.value, f.value + n.value))

    def close(self):
        if getattr(self, "_h", None):
            load_library().pfc_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- CenterShard I/O (types.hpp:29-47 layout: D x owned fp64)
    def set_shard(self, k: int, weights: np.ndarray, momentum: np.ndarray | None = None):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        m = None if momentum is None else np.ascontiguousarray(momentum, dtype=np.float64)
        _check(_lib.pfc_gpu_set_shard(self._h, k, _ptr(w), _ptr(m)), self._h)

    def get_shard(self, k: int):
        n = self.layout.owned_count(k)
        w = np.zeros((self.dim, n))
        m = np.zeros((self.dim, n))
        _check(_lib.pfc_gpu_get_shard(self._h, k, _ptr(w), _ptr(m)), self._h)
        return w, m

    def init_center_shards(self, seed: int):
        """shardsim.hpp:56-82 on the device (fp64 Box-Muller per class stream)."""
        _check(_lib.pfc_gpu_init_shards(self._h, seed), self._h)

    def device_state(self):
        w, m, rows = C.c_void_p(), C.c_void_p(), C.c_int64()
        _check(_lib.pfc_gpu_device_state(self._h, C.byref(w), C.byref(m), C.byref(rows)), self._h)
        return w.value, m.value, rows.value

    def buffers(self) -> list:
        out = []
        for k in self.local_shards:
            idx = np.zeros(self.capacity, dtype=np.int64)
            npos = C.c_int64()
            _check(_lib.pfc_gpu_get_buffers(self._h, k, _ptr(idx), C.byref(npos)), self._h)
            out.append(SampleBuffer(k, idx, npos.value))
        return out

    def stream(self) -> int:
        return _lib.pfc_gpu_stream(self._h)

    def set_step_config(self, cfg: StepConfig) -> None:
        """The reference takes a StepConfig per call: apply r / margin / filter / momentum /
        weight decay for the next steps (no-op when unchanged)."""
        cfg.margin.validate()
        c = self.cfg
        if (cfg.margin == c.margin and cfg.r == c.r and cfg.filter_threshold == c.filter_threshold
                and cfg.momentum == c.momentum and cfg.weight_decay == c.weight_decay):
            return
        sc = StepConfigC(cfg.r, cfg.margin.kind, cfg.margin.scale, cfg.margin.margin,
                         0 if cfg.filter_threshold is None else 1,
                         0.0 if cfg.filter_threshold is None else cfg.filter_threshold,
                         cfg.momentum, cfg.weight_decay, cfg.margin.m1, cfg.margin.m3)
        _check(load_library().pfc_gpu_set_step_config(self._h, C.byref(sc)), self._h)
        self.cfg = StepConfig(r=cfg.r, margin=cfg.margin, filter_threshold=cfg.filter_threshold,
                              momentum=cfg.momentum, weight_decay=cfg.weight_decay, lr=cfg.lr)
        self.capacity = load_library().pfc_gpu_capacity(self._h)

    def check_guards(self) -> int:
        """FLAG_GUARD contexts: number of guard regions a kernel overwrote (raises naming them)."""
        n = C.c_int64()
        _check(load_library().pfc_gpu_check_guards(self._h, C.byref(n)), self._h)
        return n.value

    def debug_logits(self, batch: int) -> np.ndarray:
        """Last step's logits z of this rank (FLAG_DEBUG_LOGITS): [B][local shards][cap] float32,
        -inf where the filter masked the column."""
        z = np.empty((batch, len(self.local_shards), self.capacity), dtype=np.float32)
        _check(_lib.pfc_gpu_debug_logits(self._h, _ptr(z)), self._h)
        return z

    def set_phase_timing(self, on: bool):
        _lib.pfc_gpu_set_phase_timing(self._h, 1 if on else 0)

    def phase_times(self) -> dict:
        ms = (C.c_float * 16)()
        names = (C.c_char_p * 16)()
        n = _lib.pfc_gpu_phase_times(self._h, ms, names, 16)
        return {names[i].decode(): float(ms[i]) for i in range(n)}

    def launches_per_step(self) -> int:
        return int(_lib.pfc_gpu_launches_per_step(self._h))

    def bench_inputs(self, seed: int, step: int, batch: int, x_ptr: int, labels_ptr: int):
        _check(_lib.pfc_gpu_bench_inputs(self._h, seed, step, batch, C.c_void_p(x_ptr),
                                         C.c_void_p(labels_ptr)), self._h)

    # -- steps
    def step_host(self, features_dxb: np.ndarray, labels: np.ndarray, cfg: StepConfig,
                  iteration_rng: SeededRng, out: np.ndarray | None = None) -> StepResult:
        """pfc_gpu_step on host arrays.  When features, labels and ``out`` (D x B float64,
        receives d_features) are all page-locked, the library runs its copies inside the step
        (upload overlapping the sampler, download overlapping the centre update)."""
        x = np.ascontiguousarray(features_dxb, dtype=np.float64)
        lab = np.ascontiguousarray(labels, dtype=np.int64)
        if x.ndim != 2 or x.shape[1] != lab.shape[0]:
            raise ShapeError("FeatureBatch: label count != feature columns")
        if x.shape[0] != self.dim:
            raise ShapeError(f"pfc_gpu: feature dim {x.shape[0]} != {self.dim}")
        if out is None:
            dx = np.zeros_like(x)
        else:
            if out.shape != x.shape or out.dtype != np.float64 or not out.flags.c_contiguous:
                raise ShapeError("pfc_gpu: out must be a contiguous float64 array shaped like the features")
            dx = out
        out = StepOut()
        self.set_step_config(cfg)
        args = StepArgs(iteration_rng.seed, iteration_rng.stream_id, cfg.lr, cfg.step_index)
        _check(_lib.pfc_gpu_step(self._h, _ptr(x), _ptr(lab), lab.shape[0], C.byref(args),
                                 _ptr(dx), C.byref(out)), self._h)
        tr = CollectiveTrace(out.allgather_bytes, out.reduce_scalar_bytes, out.reduce_grad_bytes,
                             out.reduce_ops)
        return StepResult(out.loss, dx, tr, [], nccl_bytes=out.nccl_bytes,
                          wire_bytes=out.wire_bytes)

    def step_features(self, features_dxb, labels, cfg: StepConfig, iteration_rng: SeededRng,
                      out=None) -> StepResult:
        """pfc_gpu_step_features: the drop-in step on a FeatureBatch already in device memory.
        features_dxb is a contiguous D x B float64 CUDA tensor, labels an int64 CUDA tensor;
        d_features go to ``out`` (D x B float64 CUDA tensor, allocated when None).  Same kernels and
        results as step_host on the same values."""
        import torch
        if not (features_dxb.is_cuda and labels.is_cuda):
            raise ContractError("step_features: features and labels must be CUDA tensors")
        x = features_dxb.contiguous()
        lab = labels.contiguous()
        if x.dtype != torch.float64 or lab.dtype != torch.int64:
            raise ShapeError("step_features: features float64, labels int64")
        if x.dim() != 2 or x.shape[1] != lab.shape[0]:
            raise ShapeError("FeatureBatch: label count != feature columns")
        if x.shape[0] != self.dim:
            raise ShapeError(f"pfc_gpu: feature dim {x.shape[0]} != {self.dim}")
        dx = torch.empty_like(x) if out is None else out
        so = StepOut()
        self.set_step_config(cfg)
        args = StepArgs(iteration_rng.seed, iteration_rng.stream_id, cfg.lr, cfg.step_index)
        torch.cuda.current_stream().synchronize()  # the library works on its own stream
        _check(_lib.pfc_gpu_step_features(self._h, x.data_ptr(), lab.data_ptr(), lab.shape[0],
                                          C.byref(args), dx.data_ptr(), C.byref(so)), self._h)
        tr = CollectiveTrace(so.allgather_bytes, so.reduce_scalar_bytes, so.reduce_grad_bytes,
                             so.reduce_ops)
        return StepResult(so.loss, dx, tr, [])

    def diagnostics(self, features_dxb: np.ndarray, labels, conflict: ConflictInfo | None = None
                    ) -> DiagnosticsSnapshot:
        """apcs / amncs of the batch against the current shards (metrics.hpp:56-146)."""
        x = np.ascontiguousarray(features_dxb, dtype=np.float64)
        lab = np.ascontiguousarray(labels, dtype=np.int64)
        if x.ndim != 2 or x.shape[1] != lab.shape[0] or x.shape[0] != self.dim:
            raise ShapeError("FeatureBatch: label count != feature columns")
        ci = si = None
        if conflict is not None:
            ci = np.ascontiguousarray(conflict.class_identity, dtype=np.int64)
            si = np.ascontiguousarray(conflict.sample_identity, dtype=np.int64)
            if ci.shape != (self.layout.num_classes,) or si.shape != lab.shape:
                raise ShapeError("ConflictInfo: identity sizes must be C and B")
        out = DiagOut()
        _check(_lib.pfc_gpu_diagnostics(self._h, _ptr(x), _ptr(lab), lab.shape[0], _ptr(ci),
                                        _ptr(si), C.byref(out)), self._h)
        return DiagnosticsSnapshot(0, out.apcs, out.amncs,
                                   out.amncs_conflicted if out.has_conflicted else None,
                                   out.amncs_hard if out.has_split else None)

    def mics(self) -> np.ndarray:
        """metrics.hpp:150-164 for the current shards: per class, the max cosine to any other."""
        out = np.zeros(self.layout.num_classes, dtype=np.float64)
        _check(_lib.pfc_gpu_mics(self._h, _ptr(out)), self._h)
        return out

    def write_shards(self, path: str, append: bool = False) -> None:
        """This rank's shard section in the reference checkpoint encoding (trainer.hpp:235-338)."""
        _check(_lib.pfc_gpu_write_shards(self._h, os.fsencode(path), 1 if append else 0), self._h)

    def read_shards(self, path: str, offset: int = 0) -> int:
        """Load a shard section at `offset`; returns the offset after it."""
        end = C.c_int64(0)
        _check(_lib.pfc_gpu_read_shards(self._h, os.fsencode(path), offset, C.byref(end)), self._h)
        return end.value

    def step_device(self, x_local_ptr: int, labels_local_ptr: int, b_local: int, dx_local_ptr: int,
                    cfg: StepConfig, iteration_rng: SeededRng, sync: bool = True):
        self.set_step_config(cfg)
        args = StepArgs(iteration_rng.seed, iteration_rng.stream_id, cfg.lr, cfg.step_index)
        out = StepOut()
        rc = _lib.pfc_gpu_step_device(self._h, C.c_void_p(x_local_ptr),
                                      C.c_void_p(labels_local_ptr), b_local, C.byref(args),
                                      C.c_void_p(dx_local_ptr), C.byref(out) if sync else None)
        _check(rc, self._h)
        return out if sync else None

    def sync(self) -> StepOut:
        out = StepOut()
        _check(_lib.pfc_gpu_sync(self._h, C.byref(out)), self._h)
        return out


def distributed_partial_step(shards: CenterShards, features_dxb: np.ndarray, labels,
                             cfg: StepConfig, iteration_rng: SeededRng) -> StepResult:
    """Drop-in for pfc::distributed_partial_step (shardsim.hpp:166-420).

    ``features_dxb``/``labels`` are the already-gathered FeatureBatch (D x B, B); ``shards`` is
    updated in place on the device; the result carries loss, the full D x B d_features, the
    reference's closed-form trace and the local shards' SampleBuffers.
    """
    cfg.margin.validate()
    diag = None
    if cfg.with_diagnostics:
        # the reference reports them for the pre-update shards (shardsim.hpp:401-417); its label
        # check (build_buffers) comes first, so validate before measuring
        lab = np.ascontiguousarray(labels, dtype=np.int64)
        bad = lab[(lab < 0) | (lab >= shards.layout.num_classes)]
        if bad.size:
            raise ContractError(f"build_buffers: label {int(np.sort(bad)[0])} outside "
                                f"[0, {shards.layout.num_classes})")
        diag = shards.diagnostics(features_dxb, lab, cfg.conflict)
        diag.iteration = cfg.step_index
    res = shards.step_host(features_dxb, labels, cfg, iteration_rng)
    res.buffers = shards.buffers()
    res.diagnostics = diag
    return res
