"""ctypes loader for the CPU oracles (TEST INFRASTRUCTURE ONLY).

Two interchangeable implementations with the same C signatures:
  * ``Oracle("port")``      -> oracle/liboracle.so, the plain-C restatement (pfc_oracle.c)
  * ``Oracle("reference")`` -> oracle/_ref/libpfc_ref.so, the unmodified reference headers
                               compiled in place (ref_shim.cpp)
Only tests/, bench.py (cpu_baseline / --impl reference) and __graft_entry__.smoke()
import this module; the product package never does.

Array conventions follow the reference value types (types.hpp:14-47): W and momentum are
the K shards' D x owned_k row-major blocks concatenated; X and dX are D x B row-major.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

STATUS = {0: "OK", 1: "ShapeError", 2: "ContractError", 3: "CapacityError", 4: "ConfigError",
          5: "NumericalError", 8: "Error", 9: "OutOfMemory"}


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS.get(status, "Error")
        self.msg = msg


class StepCfgC(C.Structure):
    _fields_ = [("r", C.c_double), ("margin_kind", C.c_int32), ("margin_scale", C.c_double),
                ("margin_m", C.c_double), ("has_filter", C.c_int32),
                ("filter_threshold", C.c_double), ("lr", C.c_double), ("momentum", C.c_double),
                ("weight_decay", C.c_double), ("step_index", C.c_int64),
                ("margin_m1", C.c_double), ("margin_m3", C.c_double)]


MARGIN_KINDS = {"plain": 0, "cosface": 1, "additive_cosine": 1, "arcface": 2,
                "additive_angular": 2, "combined": 3}  # combined: extension (pfc_oracle.c MK_COMB)


@dataclass
class OracleCfg:
    r: float = 0.1
    margin: str = "cosface"
    scale: float = 64.0
    m: float = 0.4
    filter_threshold: float | None = None
    lr: float = 0.1
    momentum: float = 0.9
    weight_decay: float = 5e-4
    step_index: int = -1
    m1: float = 1.0  # combined margin only (m = m2)
    m3: float = 0.0

    def c(self) -> StepCfgC:
        return StepCfgC(self.r, MARGIN_KINDS[self.margin], self.scale, self.m,
                        0 if self.filter_threshold is None else 1,
                        0.0 if self.filter_threshold is None else self.filter_threshold,
                        self.lr, self.momentum, self.weight_decay, self.step_index, self.m1,
                        self.m3)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libpfc_ref.so"))


class Oracle:
    def __init__(self, kind: str = "port"):
        if kind == "port":
            path, p = os.path.join(HERE, "liboracle.so"), "pfco_"
        elif kind == "reference":
            path, p = os.path.join(HERE, "_ref", "libpfc_ref.so"), "pfcr_"
        else:
            raise ValueError(kind)
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.kind = kind
        self.lib = lib = C.CDLL(path)
        self.p = p
        u64, i64, vp, dbl = C.c_uint64, C.c_int64, C.c_void_p, C.c_double
        self._f("mix64", u64, [u64])
        self._f("fnv1a", u64, [C.c_char_p, i64, u64])
        self._f("make_stream", u64, [C.c_char_p, i64, u64, u64])
        self._f("fork", u64, [u64, u64])
        self._f("draw_u64", None, [u64, u64, i64, vp])
        self._f("capacity", i64, [i64, i64, dbl])
        self._f("build_buffers", C.c_int, [i64, i64, vp, i64, dbl, u64, u64, vp, vp, C.c_char_p,
                                           C.c_int])
        self._f("init_centers", None, [i64, i64, i64, u64, vp])
        self._f("diagnostics", C.c_int, [i64, i64, i64, vp, vp, vp, i64, vp, vp, vp, vp,
                                         C.c_char_p, C.c_int])
        self._f("mics", C.c_int, [i64, i64, i64, vp, vp, C.c_char_p, C.c_int])
        self._f("step", C.c_int, [C.POINTER(StepCfgC), i64, i64, i64, vp, vp, vp, vp, i64, u64,
                                  u64, C.POINTER(dbl), vp, vp, vp, vp, vp, C.c_char_p, C.c_int])
        if kind == "port":
            self._f("step_ex", C.c_int, [C.POINTER(StepCfgC), i64, i64, i64, vp, vp, vp, vp, i64,
                                         u64, u64, C.POINTER(dbl), vp, vp, vp, vp, vp, vp,
                                         C.c_char_p, C.c_int])
        if kind == "reference":
            self._f("session_create", vp, [i64, i64, i64, u64])
            self._f("session_create_par", vp, [i64, i64, i64, u64, C.c_int])
            self._f("session_destroy", None, [vp])
            self._f("session_get", None, [vp, vp, vp])
            self._f("session_step", C.c_int, [vp, C.POINTER(StepCfgC), vp, vp, i64, u64, u64,
                                              C.POINTER(dbl), vp, C.c_char_p, C.c_int])
        else:
            self._f("bench_inputs", None, [i64, i64, i64, u64, u64, vp, vp])
            self._f("apply_margin", dbl, [dbl, C.c_int, C.c_int, dbl, dbl])
            self._f("margin_derivative", dbl, [dbl, C.c_int, C.c_int, dbl, dbl])
            self._f("apply_margin_combined", dbl, [dbl, C.c_int, dbl, dbl, dbl, dbl])
            self._f("margin_derivative_combined", dbl, [dbl, C.c_int, dbl, dbl, dbl])

    def _f(self, name, res, args):
        fn = getattr(self.lib, self.p + name)
        fn.restype = res
        fn.argtypes = args
        setattr(self, "_" + name, fn)

    # ---- rng.hpp -------------------------------------------------------------
    def mix64(self, x: int) -> int:
        return self._mix64(x)

    def fnv1a(self, s: str, h: int = 0xcbf29ce484222325) -> int:
        b = s.encode()
        return self._fnv1a(b, len(b), h)

    def make_stream(self, tag: str, a: int = 0, b: int = 0) -> int:
        t = tag.encode()
        return self._make_stream(t, len(t), a, b)

    def fork(self, stream: int, label: int) -> int:
        return self._fork(stream, label)

    def draws(self, seed: int, stream: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        self._draw_u64(seed, stream, n, _ptr(out))
        return out

    # ---- sampler.hpp ---------------------------------------------------------
    def capacity(self, C_: int, K: int, r: float) -> int:
        return self._capacity(C_, K, r)

    def build_buffers(self, C_: int, K: int, labels, r: float, seed: int, stream: int):
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        cap = self.capacity(C_, K, r)
        if cap < 0:
            raise OracleError(2, "buffer_capacity: sampling ratio must lie in (0, 1]")
        out = np.zeros((K, cap), dtype=np.int64)
        npos = np.zeros(K, dtype=np.int64)
        err = C.create_string_buffer(512)
        st = self._build_buffers(C_, K, _ptr(labels), len(labels), r, seed, stream, _ptr(out),
                                 _ptr(npos), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return out, npos

    # ---- shardsim.hpp --------------------------------------------------------
    def init_centers(self, C_: int, K: int, D: int, seed: int) -> np.ndarray:
        W = np.zeros(C_ * D, dtype=np.float64)
        self._init_centers(C_, K, D, seed, _ptr(W))
        return W

    def step(self, cfg: OracleCfg, C_: int, K: int, D: int, W: np.ndarray, M: np.ndarray,
             X: np.ndarray, labels, seed: int, stream: int, want_extra: bool = False,
             mask: np.ndarray | None = None):
        """One distributed_partial_step; W and M (shard-concatenated) are updated in place.
        ``mask`` (port only, K x B x cap bool, True = masked) replaces the filter rule."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        B = len(labels)
        assert X.shape == (D, B)
        cap = self.capacity(C_, K, cfg.r)
        dX = np.zeros((D, B), dtype=np.float64)
        bufs = np.zeros((K, max(cap, 0)), dtype=np.int64)
        npos = np.zeros(K, dtype=np.int64)
        dcent = np.zeros(K * D * max(cap, 0)) if want_extra and self.kind == "port" else None
        cosm = np.zeros(K * B * max(cap, 0)) if want_extra and self.kind == "port" else None
        loss = C.c_double(0.0)
        err = C.create_string_buffer(512)
        cc = cfg.c()
        if mask is not None:
            mk = np.ascontiguousarray(mask, dtype=np.uint8)
            assert mk.shape == (K, B, cap)
            st = self._step_ex(C.byref(cc), C_, K, D, _ptr(W), _ptr(M), _ptr(X), _ptr(labels), B,
                               seed, stream, C.byref(loss), _ptr(dX), _ptr(bufs), _ptr(npos),
                               _ptr(dcent), _ptr(cosm), _ptr(mk), err, 512)
        else:
            st = self._step(C.byref(cc), C_, K, D, _ptr(W), _ptr(M), _ptr(X), _ptr(labels), B,
                            seed, stream, C.byref(loss), _ptr(dX), _ptr(bufs), _ptr(npos),
                            _ptr(dcent), _ptr(cosm), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        out = {"loss": loss.value, "dX": dX, "buffers": bufs, "npos": npos}
        if dcent is not None:
            out["d_centers"] = dcent.reshape(K, D, cap)
            out["cos"] = cosm.reshape(K, B, cap)
        return out

    # ---- metrics.hpp (the step's diagnostics, shardsim.hpp:401-410) -------------------
    def diagnostics(self, C_: int, K: int, D: int, W: np.ndarray, X: np.ndarray, labels,
                    class_identity=None, sample_identity=None) -> dict:
        """apcs / amncs (+ conflicted / hard split) on shard-concatenated W and D x B X."""
        X = np.ascontiguousarray(X, dtype=np.float64)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        ci = None if class_identity is None else np.ascontiguousarray(class_identity, dtype=np.int64)
        si = None if sample_identity is None else np.ascontiguousarray(sample_identity, dtype=np.int64)
        out = np.zeros(4, dtype=np.float64)
        flags = np.zeros(2, dtype=np.int32)
        err = C.create_string_buffer(512)
        st = self._diagnostics(C_, K, D, _ptr(np.ascontiguousarray(W, dtype=np.float64)), _ptr(X),
                               _ptr(labels), len(labels), _ptr(ci), _ptr(si), _ptr(out),
                               _ptr(flags), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        res = {"apcs": float(out[0]), "amncs": float(out[1])}
        if flags[1]:
            res["amncs_hard"] = float(out[3])
            res["amncs_conflicted"] = float(out[2]) if flags[0] else None
        return res

    def mics(self, C_: int, K: int, D: int, W: np.ndarray) -> np.ndarray:
        """metrics.hpp:150-164: per class, the max cosine to any other class centre."""
        out = np.zeros(C_, dtype=np.float64)
        err = C.create_string_buffer(512)
        st = self._mics(C_, K, D, _ptr(np.ascontiguousarray(W, dtype=np.float64)), _ptr(out), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return out

    def bench_inputs(self, C_: int, D: int, B: int, seed: int, step: int):
        X = np.zeros((D, B), dtype=np.float64)
        labels = np.zeros(B, dtype=np.int64)
        self._bench_inputs(C_, D, B, seed, step, _ptr(X), _ptr(labels))
        return X, labels


def shard_bounds(C_: int, K: int):
    """ShardLayout (sampler.hpp:16-33): [(owned_begin, owned_end)] per shard."""
    blk = (C_ + K - 1) // K
    return [(min(k * blk, C_), min((k + 1) * blk, C_)) for k in range(K)]


def shards_to_rows(W: np.ndarray, C_: int, K: int, D: int) -> np.ndarray:
    """Shard-concatenated D x owned blocks -> C x D row-major (class rows)."""
    out = np.empty((C_, D), dtype=W.dtype)
    off = 0
    for lo, hi in shard_bounds(C_, K):
        n = hi - lo
        out[lo:hi] = W[off:off + D * n].reshape(D, n).T
        off += D * n
    return out


def rows_to_shards(R: np.ndarray, C_: int, K: int, D: int) -> np.ndarray:
    parts = [np.ascontiguousarray(R[lo:hi].T).ravel() for lo, hi in shard_bounds(C_, K)]
    return np.concatenate(parts)


def fnv64(a) -> str:
    """FNV-1a-64 over int64 little-endian bytes (the sampler checksum of SURVEY.md Appendix B)."""
    h = 0xcbf29ce484222325
    for byte in np.ascontiguousarray(a, dtype="<i8").tobytes():
        h ^= byte
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
