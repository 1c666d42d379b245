"""ctypes binding of libmlstm.so (include/mlstm.h).  Argument marshalling only: every step of the
training path runs in the library's CUDA kernels.  There is no CPU fallback -- if the library is
missing or no sm_100a device is present the calls raise.

The function names mirror the C ABI (mlstm_init, mlstm_train_step, ...).  ``MLSTM`` is a small
convenience owner of one context: it allocates the workspace with torch (device memory) and
passes torch's current stream (PyTorch is used for memory, streams and process groups only).
"""
from __future__ import annotations

import ctypes
import math
import os
import re

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MLSTM_LIB") or os.path.join(HERE, "libmlstm.so")  # MLSTM_LIB: A/B experiments
HEADER = os.path.join(os.path.dirname(HERE), "include", "mlstm.h")
HEADERS = [HEADER, os.path.join(os.path.dirname(HERE), "include", "mlstm_data.h")]

MLSTM_OK, MLSTM_EINVAL, MLSTM_ECUDA, MLSTM_ENCCL, MLSTM_ENOMEM, MLSTM_ESTATE, MLSTM_EDIVERGED = range(7)
MLSTM_FP32, MLSTM_MIXED = 0, 1
MLSTM_LR_NONE, MLSTM_LR_LINEAR, MLSTM_LR_SQRT = 0, 1, 2
MLSTM_ASYNC = 1
MLSTM_SLOT_TRAIN, MLSTM_SLOT_EVAL = 0, 1
STATUS_NAMES = ["OK", "EINVAL", "ECUDA", "ENCCL", "ENOMEM", "ESTATE", "EDIVERGED"]


class MlstmConfig(ctypes.Structure):
    _fields_ = [
        ("hidden", ctypes.c_int32), ("embed", ctypes.c_int32), ("vocab", ctypes.c_int32),
        ("seq_len", ctypes.c_int32), ("batch", ctypes.c_int32), ("micro_batch", ctypes.c_int32),
        ("precision", ctypes.c_int32), ("weight_norm", ctypes.c_int32), ("seed", ctypes.c_uint64),
        ("lr0", ctypes.c_double), ("decay_iters", ctypes.c_int64), ("beta1", ctypes.c_double),
        ("beta2", ctypes.c_double), ("eps", ctypes.c_double), ("scale_init", ctypes.c_float),
        ("scale_min", ctypes.c_float), ("scale_max", ctypes.c_float),
        ("scale_growth_interval", ctypes.c_int32), ("diverge_patience", ctypes.c_int32),
        ("recurrence", ctypes.c_int32),
    ]


class MlstmStepResult(ctypes.Structure):
    _fields_ = [
        ("loss_nats", ctypes.c_double), ("bpc", ctypes.c_double), ("lr", ctypes.c_double),
        ("loss_scale", ctypes.c_float), ("skipped", ctypes.c_int32), ("step", ctypes.c_int64),
        ("applied", ctypes.c_int64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class MlstmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"mlstm {STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")
        self.status = status


_lib = None
_P = ctypes.POINTER
_vp, _u8p, _fp, _dp = ctypes.c_void_p, _P(ctypes.c_uint8), _P(ctypes.c_float), _P(ctypes.c_double)
_i32p, _i64p = _P(ctypes.c_int32), _P(ctypes.c_int64)

_SIGS = {
    "mlstm_default_config": (None, [_P(MlstmConfig)]),
    "mlstm_param_count": (ctypes.c_int64, [_P(MlstmConfig)]),
    "mlstm_workspace_bytes": (ctypes.c_size_t, [_P(MlstmConfig)]),
    "mlstm_nccl_unique_id": (ctypes.c_int, [_u8p]),
    "mlstm_init": (ctypes.c_int, [_P(MlstmConfig), _vp, ctypes.c_size_t, _vp, _u8p, ctypes.c_int, ctypes.c_int,
                                  _P(_vp)]),
    "mlstm_train_step": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_uint32, _P(MlstmStepResult)]),
    "mlstm_train_step_host": (ctypes.c_int, [_vp, _u8p, _u8p, _P(MlstmStepResult)]),
    "mlstm_eval": (ctypes.c_int, [_vp, _vp, ctypes.c_int32, _vp, _dp, _i64p, _dp]),
    "mlstm_lr_at": (ctypes.c_double, [ctypes.c_double, ctypes.c_int64, ctypes.c_int64]),
    "mlstm_scale_lr": (ctypes.c_double, [ctypes.c_double, ctypes.c_int, ctypes.c_int64, ctypes.c_int64]),
    "mlstm_bpc_from_nats": (ctypes.c_double, [ctypes.c_double]),
    "mlstm_get_params": (ctypes.c_int, [_vp, _fp]),
    "mlstm_set_params": (ctypes.c_int, [_vp, _fp]),
    "mlstm_get_grads": (ctypes.c_int, [_vp, _fp]),
    "mlstm_get_state": (ctypes.c_int, [_vp, ctypes.c_int, _fp, _fp]),
    "mlstm_set_state": (ctypes.c_int, [_vp, ctypes.c_int, _fp, _fp]),
    "mlstm_get_opt_state": (ctypes.c_int, [_vp, _fp, _fp, _i64p, _fp, _i32p, _i64p]),
    "mlstm_set_opt_state": (ctypes.c_int, [_vp, _fp, _fp, ctypes.c_int64, ctypes.c_float, ctypes.c_int32,
                                           ctypes.c_int64]),
    "mlstm_debug_dump": (ctypes.c_int, [_vp, ctypes.c_char_p, _fp, ctypes.c_size_t]),
    "mlstm_check_overflow": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int, _i32p]),
    "mlstm_profile_enable": (ctypes.c_int, [_vp, ctypes.c_int]),
    "mlstm_phase_times": (ctypes.c_int, [_vp, _dp, _i32p, _i32p]),
    "mlstm_phase_name": (ctypes.c_char_p, [ctypes.c_int]),
    "mlstm_launches_per_step": (ctypes.c_int32, [_vp]),
    "mlstm_recurrence_kind": (ctypes.c_int32, [_vp]),
    "mlstm_gemm_bench": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, _dp]),
    "mlstm_trace_enable": (ctypes.c_int, [ctypes.c_int]),
    "mlstm_trace_read": (ctypes.c_int, [_P(ctypes.c_uint64), ctypes.c_int, _i32p]),
    # data pipeline (include/mlstm_data.h)
    "mlstm_corpus_create": (ctypes.c_int, [_u8p, _P(ctypes.c_int64), ctypes.c_int64, ctypes.c_uint64,
                                           _P(ctypes.c_void_p)]),
    "mlstm_corpus_split_sizes": (ctypes.c_int, [_vp, _P(ctypes.c_int64)]),
    "mlstm_corpus_destroy": (None, [_vp]),
    "mlstm_loader_create": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.c_uint64, _P(ctypes.c_void_p)]),
    "mlstm_loader_num_shards": (ctypes.c_int64, [_vp]),
    "mlstm_loader_shard": (ctypes.c_int, [_vp, ctypes.c_int64, _u8p, ctypes.c_int64, _P(ctypes.c_int64)]),
    "mlstm_loader_next": (ctypes.c_int, [_vp, _u8p, _u8p, _u8p, _i32p]),
    "mlstm_heldout_bpc": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _dp, _i64p, _dp]),
    "mlstm_loader_rewind": (ctypes.c_int, [_vp]),
    "mlstm_loader_destroy": (None, [_vp]),
    "mlstm_last_error": (ctypes.c_char_p, []),
    "mlstm_destroy": (None, [_vp]),
    "mlstm_sync": (ctypes.c_int, [_vp]),
    "mlstm_allreduce_plan": (ctypes.c_int, [_P(MlstmConfig), ctypes.c_int32, _i64p, ctypes.c_int32, _i32p]),
}


def lib():
    """Loads libmlstm.so (in-tree).  Raises if it has not been built -- no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_1808_01371_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def header_functions():
    """Names of the functions include/*.h declare (mlstm.h: the step; mlstm_data.h: the data pipeline)."""
    names = set()
    for h in HEADERS:
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        names |= set(re.findall(r"\b(mlstm_[a-z_0-9]+)\s*\(", src))
    return sorted(names)


def _check(status):
    if status != MLSTM_OK:
        raise MlstmError(status, lib().mlstm_last_error().decode())


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a, typ=ctypes.c_float):
    return a.ctypes.data_as(ctypes.POINTER(typ))


# ------------------------------------------------------------------ same names as the C ABI
def mlstm_default_config(**overrides) -> MlstmConfig:
    cfg = MlstmConfig()
    lib().mlstm_default_config(ctypes.byref(cfg))
    for k, v in overrides.items():
        if not hasattr(cfg, k):
            raise KeyError(k)
        setattr(cfg, k, v)
    return cfg


def mlstm_param_count(cfg: MlstmConfig) -> int:
    return int(lib().mlstm_param_count(ctypes.byref(cfg)))


def mlstm_workspace_bytes(cfg: MlstmConfig) -> int:
    n = int(lib().mlstm_workspace_bytes(ctypes.byref(cfg)))
    if n == 0:
        raise MlstmError(MLSTM_EINVAL, lib().mlstm_last_error().decode())
    return n


def mlstm_allreduce_plan(cfg: MlstmConfig, world: int) -> list[tuple[int, int, int]]:
    """Bucket plan of the gradient allreduce: [(offset, count, after)] in reduction order."""
    n = ctypes.c_int32()
    out = np.zeros((16, 3), dtype=np.int64)
    _check(lib().mlstm_allreduce_plan(ctypes.byref(cfg), world, out.ctypes.data_as(_i64p), 16, ctypes.byref(n)))
    return [tuple(int(v) for v in row) for row in out[: n.value]]


def mlstm_nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().mlstm_nccl_unique_id(buf))
    return bytes(buf)


def mlstm_init(cfg, workspace_ptr: int, workspace_bytes: int, stream_ptr: int, nccl_id: bytes | None,
               rank: int, world: int):
    ctx = ctypes.c_void_p()
    idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
    _check(lib().mlstm_init(ctypes.byref(cfg), ctypes.c_void_p(workspace_ptr), workspace_bytes,
                            ctypes.c_void_p(stream_ptr), idbuf, rank, world, ctypes.byref(ctx)))
    return ctx


def mlstm_train_step(ctx, bytes_ptr: int, reset_ptr: int | None = None, flags: int = 0) -> MlstmStepResult:
    out = MlstmStepResult()
    _check(lib().mlstm_train_step(ctx, ctypes.c_void_p(bytes_ptr), ctypes.c_void_p(reset_ptr or 0), flags,
                                  ctypes.byref(out)))
    return out


def mlstm_train_step_host(ctx, bytes_host: np.ndarray, reset_host: np.ndarray | None = None) -> MlstmStepResult:
    out = MlstmStepResult()
    b = np.ascontiguousarray(bytes_host, dtype=np.uint8)
    r = None if reset_host is None else np.ascontiguousarray(reset_host, dtype=np.uint8)
    _check(lib().mlstm_train_step_host(ctx, _ptr(b, ctypes.c_uint8), None if r is None else _ptr(r, ctypes.c_uint8),
                                       ctypes.byref(out)))
    return out


def mlstm_eval(ctx, bytes_ptr: int, Be: int, reset_ptr: int | None = None):
    nats, tok, bpc = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
    _check(lib().mlstm_eval(ctx, ctypes.c_void_p(bytes_ptr), Be, ctypes.c_void_p(reset_ptr or 0),
                            ctypes.byref(nats), ctypes.byref(tok), ctypes.byref(bpc)))
    return nats.value, tok.value, bpc.value


def mlstm_lr_at(lr0: float, it: int, decay_iters: int) -> float:
    return lib().mlstm_lr_at(lr0, it, decay_iters)


def mlstm_scale_lr(base_lr: float, rule: int, batch: int, ref_batch: int = 128) -> float:
    return lib().mlstm_scale_lr(base_lr, rule, batch, ref_batch)


def mlstm_bpc_from_nats(nats: float) -> float:
    return lib().mlstm_bpc_from_nats(nats)


def mlstm_gemm_bench(engine: int, M: int, N: int, K: int, bn: int = 0, iters: int = 20) -> float:
    ms = ctypes.c_double()
    _check(lib().mlstm_gemm_bench(engine, M, N, K, bn, iters, ctypes.byref(ms)))
    return ms.value


def mlstm_trace_enable(capacity: int) -> None:
    _check(lib().mlstm_trace_enable(capacity))


def mlstm_trace_read(capacity: int = 1 << 20) -> np.ndarray:
    out = np.zeros((capacity, 12), dtype=np.uint64)
    n = ctypes.c_int32()
    _check(lib().mlstm_trace_read(out.ctypes.data_as(_P(ctypes.c_uint64)), capacity, ctypes.byref(n)))
    return out[: n.value]


def mlstm_destroy(ctx):
    lib().mlstm_destroy(ctx)


class MLSTM:
    """Owns one context on the current CUDA device (one process per GPU)."""

    def __init__(self, cfg: MlstmConfig, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("MLSTM needs a CUDA device (sm_100a); there is no CPU fallback")
        self.cfg = cfg
        self.B, self.T, self.h = cfg.batch, cfg.seq_len, cfg.hidden
        self.P = mlstm_param_count(cfg)
        self.ws_bytes = mlstm_workspace_bytes(cfg)
        self.workspace = torch.empty(self.ws_bytes, dtype=torch.uint8, device="cuda")
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.ctx = mlstm_init(cfg, self.workspace.data_ptr(), self.ws_bytes, self.stream.cuda_stream, nccl_id,
                              rank, world)
        self.rank, self.world = rank, world

    def close(self):
        if getattr(self, "ctx", None):
            mlstm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # training / evaluation -------------------------------------------------------------
    def train_step(self, bytes_dev, reset_dev=None, flags: int = 0) -> dict:
        """bytes_dev: torch uint8 CUDA tensor [B, T+1]; reset_dev: uint8 CUDA [B] or None."""
        assert bytes_dev.dtype.itemsize == 1 and bytes_dev.is_cuda and bytes_dev.is_contiguous()
        assert tuple(bytes_dev.shape) == (self.B, self.T + 1)
        r = mlstm_train_step(self.ctx, bytes_dev.data_ptr(), None if reset_dev is None else reset_dev.data_ptr(),
                             flags)
        return r.as_dict()

    def train_step_async(self, bytes_dev, reset_dev=None):
        """Enqueues one step with MLSTM_ASYNC; returns the result struct the library fills at the
        next synchronising call (sync(), or a train_step without the flag)."""
        assert bytes_dev.dtype.itemsize == 1 and bytes_dev.is_cuda and bytes_dev.is_contiguous()
        assert tuple(bytes_dev.shape) == (self.B, self.T + 1)
        out = MlstmStepResult()
        self._pending = getattr(self, "_pending", []) + [out]  # keeps *out alive until delivered
        _check(lib().mlstm_train_step(self.ctx, ctypes.c_void_p(bytes_dev.data_ptr()),
                                      ctypes.c_void_p(0 if reset_dev is None else reset_dev.data_ptr()),
                                      MLSTM_ASYNC, ctypes.byref(out)))
        return out

    def sync(self) -> None:
        """mlstm_sync: delivers every outstanding async result (raises MlstmError on divergence)."""
        try:
            _check(lib().mlstm_sync(self.ctx))
        finally:
            self._pending = []

    def train_step_host(self, bytes_host, reset_host=None) -> dict:
        assert np.asarray(bytes_host).shape == (self.B, self.T + 1)
        return mlstm_train_step_host(self.ctx, bytes_host, reset_host).as_dict()

    def eval(self, bytes_dev, reset_dev=None):
        Be = int(bytes_dev.shape[0])
        return mlstm_eval(self.ctx, bytes_dev.data_ptr(), Be, None if reset_dev is None else reset_dev.data_ptr())

    # state access ----------------------------------------------------------------------
    def get_params(self) -> np.ndarray:
        out = np.empty(self.P, dtype=np.float32)
        _check(lib().mlstm_get_params(self.ctx, _ptr(out)))
        return out

    def set_params(self, flat) -> None:
        a = _f32(flat)
        assert a.size == self.P
        _check(lib().mlstm_set_params(self.ctx, _ptr(a)))

    def get_grads(self) -> np.ndarray:
        out = np.empty(self.P, dtype=np.float32)
        _check(lib().mlstm_get_grads(self.ctx, _ptr(out)))
        return out

    def get_state(self, slot: int = MLSTM_SLOT_TRAIN):
        h = np.empty((self.B, self.h), dtype=np.float32)
        c = np.empty((self.B, self.h), dtype=np.float32)
        _check(lib().mlstm_get_state(self.ctx, slot, _ptr(h), _ptr(c)))
        return h, c

    def set_state(self, h, c, slot: int = MLSTM_SLOT_TRAIN):
        hh, cc = _f32(h), _f32(c)
        _check(lib().mlstm_set_state(self.ctx, slot, _ptr(hh), _ptr(cc)))

    def get_opt_state(self):
        m = np.empty(self.P, dtype=np.float32)
        v = np.empty(self.P, dtype=np.float32)
        tau, alpha, clean, it = ctypes.c_int64(), ctypes.c_float(), ctypes.c_int32(), ctypes.c_int64()
        _check(lib().mlstm_get_opt_state(self.ctx, _ptr(m), _ptr(v), ctypes.byref(tau), ctypes.byref(alpha),
                                         ctypes.byref(clean), ctypes.byref(it)))
        return {"m": m, "v": v, "tau": tau.value, "alpha": alpha.value, "clean": clean.value, "it": it.value}

    def set_opt_state(self, m=None, v=None, tau=0, alpha=65536.0, clean=0, it=0):
        mm = None if m is None else _f32(m)
        vv = None if v is None else _f32(v)
        _check(lib().mlstm_set_opt_state(self.ctx, None if mm is None else _ptr(mm), None if vv is None else _ptr(vv),
                                         tau, alpha, clean, it))

    def debug_dump(self, name: str, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float32)
        _check(lib().mlstm_debug_dump(self.ctx, name.encode(), _ptr(out), count))
        return out

    def check_overflow(self, tensor) -> bool:
        import torch
        dtype = {torch.float16: 0, torch.float32: 1}[tensor.dtype]
        flag = ctypes.c_int32()
        _check(lib().mlstm_check_overflow(self.ctx, ctypes.c_void_p(tensor.data_ptr()), tensor.numel(), dtype,
                                          ctypes.byref(flag)))
        return bool(flag.value)

    def profile(self, enable: bool = True):
        _check(lib().mlstm_profile_enable(self.ctx, int(enable)))

    def phase_times(self) -> dict:
        ms = (ctypes.c_double * 16)()
        ln = (ctypes.c_int32 * 16)()
        n = ctypes.c_int32()
        _check(lib().mlstm_phase_times(self.ctx, ms, ln, ctypes.byref(n)))
        return {lib().mlstm_phase_name(i).decode(): (ms[i], ln[i]) for i in range(n.value)}

    def uses_recur(self) -> bool:
        """True when the recurrence runs on the persistent dataflow kernels (mlstm_recurrence_kind)."""
        return lib().mlstm_recurrence_kind(self.ctx) in (1, 3)

    def launches_per_step(self) -> int:
        n = lib().mlstm_launches_per_step(self.ctx)
        if n < 0:
            _check(MLSTM_ECUDA)
        return int(n)


# ------------------------------------------------------------------ data pipeline (mlstm_data.h)
MLSTM_SPLIT_TRAIN, MLSTM_SPLIT_VAL, MLSTM_SPLIT_TEST = 0, 1, 2
MLSTM_SHARDS_TRAIN, MLSTM_SHARDS_EVAL = 0, 1


class Corpus:
    """Records (list of bytes) -> the 1000:1:1 split held by the library."""

    def __init__(self, records, seed: int = 0x5EED):
        self.h = None
        data = np.frombuffer(b"".join(records), dtype=np.uint8) if records else np.zeros(0, np.uint8)
        data = np.ascontiguousarray(data) if data.size else np.zeros(1, np.uint8)
        offs = np.zeros(len(records) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(r) for r in records])
        h = ctypes.c_void_p()
        _check(lib().mlstm_corpus_create(_ptr(data, ctypes.c_uint8), offs.ctypes.data_as(_P(ctypes.c_int64)), len(records),
                                         seed, ctypes.byref(h)))
        self.h = h

    def split_sizes(self):
        out = (ctypes.c_int64 * 3)()
        _check(lib().mlstm_corpus_split_sizes(self.h, out))
        return tuple(out)

    def close(self):
        if self.h:
            lib().mlstm_corpus_destroy(self.h)
            self.h = None

    __del__ = close


class Loader:
    """Shard-contiguous TBTT minibatches of one split: next() -> (bytes [B][T+1], reset [B])
    or None at the end of the epoch."""

    def __init__(self, corpus: Corpus, split: int, kind: int, B: int, T: int, seed: int = 0x5EED):
        self.h = None
        h = ctypes.c_void_p()
        _check(lib().mlstm_loader_create(corpus.h, split, kind, B, T, seed, ctypes.byref(h)))
        self.h, self.B, self.T = h, B, T

    def num_shards(self) -> int:
        return lib().mlstm_loader_num_shards(self.h)

    def shard(self, i: int) -> bytes:
        n = ctypes.c_int64()
        _check(lib().mlstm_loader_shard(self.h, i, None, 0, ctypes.byref(n)))
        buf = np.zeros(max(1, n.value), dtype=np.uint8)
        _check(lib().mlstm_loader_shard(self.h, i, _ptr(buf, ctypes.c_uint8), n.value, ctypes.byref(n)))
        return buf[:n.value].tobytes()

    def next(self):
        """(bytes [B, T+1], reset [B], valid [B]) or None at the end of the epoch."""
        by = np.zeros((self.B, self.T + 1), dtype=np.uint8)
        rs = np.zeros(self.B, dtype=np.uint8)
        ok = np.zeros(self.B, dtype=np.uint8)
        end = ctypes.c_int32()
        _check(lib().mlstm_loader_next(self.h, _ptr(by, ctypes.c_uint8), _ptr(rs, ctypes.c_uint8),
                                       _ptr(ok, ctypes.c_uint8), ctypes.byref(end)))
        return None if end.value else (by, rs, ok)

    def rewind(self):
        _check(lib().mlstm_loader_rewind(self.h))

    def __iter__(self):
        while True:
            b = self.next()
            if b is None:
                return
            yield b

    def close(self):
        if self.h:
            lib().mlstm_loader_destroy(self.h)
            self.h = None

    __del__ = close


def heldout_bpc(model, loader: Loader, max_batches: int | None = None) -> float:
    """Held-out BPC over one epoch of an evaluation loader: mlstm_heldout_bpc (the library runs
    every window through the evaluation forward with the loader's reset masks and accumulates)."""
    nats, tok, bpc = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
    _check(lib().mlstm_heldout_bpc(model.ctx, loader.h, -1 if max_batches is None else max_batches,
                                   ctypes.byref(nats), ctypes.byref(tok), ctypes.byref(bpc)))
    return bpc.value


def cell_features(model, texts):
    """Frozen-feature transfer: the final cell state c_T of each text after a
    forward-only pass from a zero state (mlstm_eval over consecutive T-byte windows with the state
    carried, reset at the first window).  texts: list of equal-length byte strings of
    1 + k*T bytes, at most `batch` of them per call.  Returns float32 [len(texts), h]."""
    import torch
    n, T = len(texts), model.T
    L = len(texts[0])
    if n > model.B or any(len(t) != L for t in texts) or (L - 1) % T or L < T + 1:
        raise ValueError("texts: <= batch strings of equal length 1 + k*T")
    arr = np.frombuffer(b"".join(texts), dtype=np.uint8).reshape(n, L)
    reset = torch.ones(n, dtype=torch.uint8, device="cuda")
    for k in range((L - 1) // T):
        window = torch.from_numpy(np.ascontiguousarray(arr[:, k * T: k * T + T + 1])).cuda()
        model.eval(window, reset if k == 0 else None)
    return model.get_state(MLSTM_SLOT_EVAL)[1][:n].copy()
