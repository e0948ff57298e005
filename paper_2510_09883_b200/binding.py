"""ctypes binding of ``libdelta.so`` (include/delta.h) — argument marshalling only.

Every step of the decode path runs in the library's sm_100a kernels.  There is no CPU or
PyTorch fallback: if the shared library is missing this module raises on load.
PyTorch provides device memory, streams and process groups (plumbing).
"""
from __future__ import annotations

import ctypes
import os
import re
from dataclasses import dataclass, field

_HERE = os.path.dirname(os.path.abspath(__file__))
# DELTA_LIB_PATH selects an instrumented build of the SAME sources (make trace) for latency
# analysis; the product library is the in-tree libdelta.so.
LIB_PATH = os.environ.get("DELTA_LIB_PATH") or os.path.join(_HERE, "libdelta.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "delta.h")

DELTA_BF16, DELTA_FP32 = 0, 1
ROLE_FULL, ROLE_SELECT, ROLE_SPARSE, ROLE_QUEST, ROLE_RAAS = 0, 1, 2, 3, 4
POLICY_DELTA, POLICY_QUEST, POLICY_RAAS = 0, 1, 2
STATUS = {0: "OK", 1: "CONFIG", 2: "USAGE", 3: "NUMERIC", 4: "CAPACITY", 5: "CUDA", 6: "NCCL"}


class DeltaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"DELTA_ERR_{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Config(ctypes.Structure):
    _fields_ = [
        ("num_layers", ctypes.c_int32), ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32), ("max_batch", ctypes.c_int32), ("max_seq_len", ctypes.c_int32),
        ("page_size", ctypes.c_int32), ("num_phys_pages", ctypes.c_int32), ("num_full_prefix", ctypes.c_int32),
        ("num_select_layers", ctypes.c_int32), ("select_layers", ctypes.POINTER(ctypes.c_int32)),
        ("budget_k", ctypes.c_int32), ("n_sink", ctypes.c_int32), ("n_window", ctypes.c_int32),
        ("select_block", ctypes.c_int32), ("kv_dtype", ctypes.c_int), ("softmax_scale", ctypes.c_float),
        ("shard_world", ctypes.c_int32), ("shard_rank", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
        ("policy", ctypes.c_int32), ("det_chunks", ctypes.c_int32),
    ]


class _Buffers(ctypes.Structure):
    _fields_ = [("kv_pool", ctypes.c_void_p), ("block_table", ctypes.c_void_p),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t)]


_lib = None


def load_library() -> ctypes.CDLL:
    """Load libdelta.so; raise if it is not built (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                           "there is no CPU/PyTorch fallback for the DELTA decode path")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, st = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int
    L.delta_query_sizes.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(ctypes.c_size_t),
                                    ctypes.POINTER(ctypes.c_size_t)]
    L.delta_query_sizes.restype = st
    L.delta_create.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(_Buffers), ctypes.POINTER(vp)]
    L.delta_create.restype = st
    L.delta_set_seq_lens.argtypes = [vp, i32, i32, ctypes.POINTER(i32), vp]
    L.delta_set_seq_lens.restype = st
    L.delta_append_kv.argtypes = [vp, i32, i32, i32, vp, vp, vp]
    L.delta_append_kv.restype = st
    L.delta_decode_layer.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    L.delta_decode_layer.restype = st
    L.delta_append_decode_layer.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp]
    L.delta_append_decode_layer.restype = st
    L.delta_select.argtypes = [vp, i32, i32, vp, vp, vp, vp]
    L.delta_select.restype = st
    L.delta_decode_step.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp]
    L.delta_decode_step.restype = st
    L.delta_decode_step_host.argtypes = [vp, i32, vp, vp, vp, vp, vp]
    L.delta_decode_step_host.restype = st
    L.delta_get_error.argtypes = [vp, vp, ctypes.POINTER(st)]
    L.delta_get_error.restype = st
    L.delta_layer_role.argtypes = [vp, i32]
    L.delta_layer_role.restype = st
    L.delta_governing_layer.argtypes = [vp, i32]
    L.delta_governing_layer.restype = i32
    L.delta_plan_capacity.argtypes = [vp]
    L.delta_plan_capacity.restype = i32
    L.delta_last_error_message.argtypes = [vp]
    L.delta_last_error_message.restype = ctypes.c_char_p
    L.delta_version.argtypes = []
    L.delta_version.restype = ctypes.c_char_p
    L.delta_destroy.argtypes = [vp]
    L.delta_destroy.restype = st
    L.delta_kernels_launched.argtypes = [vp]
    L.delta_kernels_launched.restype = ctypes.c_uint64
    L.delta_set_tuning.argtypes = [vp, ctypes.c_char_p, i32]
    L.delta_set_tuning.restype = st
    L.delta_layer_kernel_name.argtypes = [vp, i32, i32]
    L.delta_layer_kernel_name.restype = ctypes.c_char_p
    L.delta_graph_captures.argtypes = [vp]
    L.delta_graph_captures.restype = ctypes.c_uint64
    L.delta_read_bandwidth_probe.argtypes = [vp, ctypes.c_size_t, vp, vp]
    L.delta_read_bandwidth_probe.restype = st
    L.delta_set_nccl_library.argtypes = [ctypes.c_char_p]
    L.delta_set_nccl_library.restype = st
    L.delta_nccl_get_unique_id.argtypes = [vp]
    L.delta_nccl_get_unique_id.restype = st
    L.delta_shard_range.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.delta_shard_range.restype = st
    L.delta_shard_exchange_buffers.argtypes = [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(vp),
                                               ctypes.POINTER(ctypes.c_size_t)]
    L.delta_shard_exchange_buffers.restype = st
    L.delta_shard_merge.argtypes = [vp, i32, i32, vp, vp, vp]
    L.delta_shard_merge.restype = st
    L.delta_shard_select_merge.argtypes = [vp, i32, i32, vp, vp, vp]
    L.delta_shard_select_merge.restype = st
    L.delta_quest_build_reps.argtypes = [vp, i32, i32, vp]
    L.delta_quest_build_reps.restype = st
    L.delta_copy_plan.argtypes = [vp, i32, i32, vp, vp, vp]
    L.delta_copy_plan.restype = st
    L.delta_attention_recall.argtypes = [vp, i32, i32, vp, vp, vp]
    L.delta_attention_recall.restype = st
    L.delta_raas_reset.argtypes = [vp, i32, i32, vp]
    L.delta_raas_reset.restype = st
    L.delta_prefill.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp]
    L.delta_prefill.restype = st
    L.delta_workspace_region.argtypes = [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_size_t)]
    L.delta_workspace_region.restype = st
    _lib = L
    return L


def declared_functions() -> list[str]:
    """Function names declared in include/delta.h (the boundary)."""
    src = open(HEADER_PATH).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(delta_[a-z_0-9]+)\s*\(", src)))


@dataclass
class DeltaConfig:
    """Problem statement of the method: schedule, budget, paged layout (include/delta.h)."""
    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    max_batch: int
    max_seq_len: int
    num_full_prefix: int
    select_layers: list = field(default_factory=list)
    budget_k: int = 2048
    n_sink: int = 4
    n_window: int = 32
    select_block: int = 16
    kv_dtype: int = DELTA_BF16
    softmax_scale: float = 0.0
    page_size: int = 16
    num_phys_pages: int = 0
    shard_world: int = 1
    shard_rank: int = 0
    nccl_id: bytes | None = None   # 128 bytes from nccl_unique_id() (rank 0), or None
    policy: int = POLICY_DELTA
    det_chunks: int = 0            # R21 fixed chunks (bitwise identical results for every W | C)

    def to_c(self):
        arr = (ctypes.c_int32 * max(1, len(self.select_layers)))(*self.select_layers)
        nid = ctypes.create_string_buffer(self.nccl_id, 128) if self.nccl_id else None
        c = _Config(self.num_layers, self.num_q_heads, self.num_kv_heads, self.head_dim, self.max_batch,
                    self.max_seq_len, self.page_size, self.num_phys_pages, self.num_full_prefix,
                    len(self.select_layers), arr, self.budget_k, self.n_sink, self.n_window, self.select_block,
                    self.kv_dtype, self.softmax_scale, self.shard_world, self.shard_rank,
                    ctypes.cast(nid, ctypes.c_void_p) if nid is not None else None, self.policy,
                    self.det_chunks)
        return c, (arr, nid)  # keep alive

    @property
    def max_pages(self) -> int:
        return -(-self.max_seq_len // self.page_size)

    @property
    def phys_pages(self) -> int:
        return self.num_phys_pages or self.max_batch * self.max_pages


def _check(st: int, handle=None):
    if st != 0:
        msg = load_library().delta_last_error_message(handle)
        raise DeltaError(st, msg.decode() if msg else "")


def query_sizes(cfg: DeltaConfig) -> tuple[int, int]:
    L = load_library()
    c, _keep = cfg.to_c()
    pb, wb = ctypes.c_size_t(), ctypes.c_size_t()
    _check(L.delta_query_sizes(ctypes.byref(c), ctypes.byref(pb), ctypes.byref(wb)))
    return pb.value, wb.value


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId from rank 0 (to broadcast with torch.distributed)."""
    import os
    try:
        import nvidia.nccl  # the copy torch uses
        path = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        _check(load_library().delta_set_nccl_library(path.encode()))
    except ImportError:
        pass
    buf = ctypes.create_string_buffer(128)
    _check(load_library().delta_nccl_get_unique_id(buf))
    return buf.raw


def shard_range(cfg: DeltaConfig) -> tuple[int, int]:
    """[page_lo, page_hi) of every sequence held by rank cfg.shard_rank (host-only)."""
    c, _keep = cfg.to_c()
    lo, hi = ctypes.c_int32(), ctypes.c_int32()
    _check(load_library().delta_shard_range(ctypes.byref(c), ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def read_bandwidth_probe(buf, sink, stream=None):
    """Pure-read roofline kernel (measurement utility): streams the device
    tensor `buf` once; `sink` is a 1-element fp32 device tensor."""
    assert buf.is_cuda and sink.is_cuda and sink.dtype.is_floating_point
    _check(load_library().delta_read_bandwidth_probe(buf.data_ptr(), buf.numel() * buf.element_size(),
                                                      sink.data_ptr(), _stream(stream)))


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class DeltaStack:
    """One handle of the DELTA decode-attention stack over caller-owned torch buffers."""

    def __init__(self, cfg: DeltaConfig, kv_pool, block_table, workspace):
        """kv_pool: [L][phys_pages][g][2][P][d] (K rows then V rows per (page, head))."""
        self.cfg = cfg
        self.lib = load_library()
        self.kv_pool, self.block_table, self.workspace = kv_pool, block_table, workspace
        c, self._keep = cfg.to_c()
        b = _Buffers(kv_pool.data_ptr(), block_table.data_ptr(), workspace.data_ptr(),
                     workspace.numel() * workspace.element_size())
        h = ctypes.c_void_p()
        _check(self.lib.delta_create(ctypes.byref(c), ctypes.byref(b), ctypes.byref(h)))
        self.h = h
        import os
        tune = os.environ.get("DELTA_TUNE", "")  # experiment knobs (tools/), "key=value,..."
        for kv in filter(None, tune.split(",")):
            k, v = kv.split("=")
            self.set_tuning(k.strip(), int(v))

    def set_tuning(self, key: str, value: int):
        """Kernel-variant knob for experiments (delta_set_tuning)."""
        _check(self.lib.delta_set_tuning(self.h, key.encode(), value), self.h)

    @property
    def k_pool(self):
        """View [L][phys_pages][g][P][d] of the key rows of kv_pool."""
        return self.kv_pool[:, :, :, 0]

    @property
    def v_pool(self):
        """View [L][phys_pages][g][P][d] of the value rows of kv_pool."""
        return self.kv_pool[:, :, :, 1]

    @classmethod
    def allocate(cls, cfg: DeltaConfig, block_table, device="cuda"):
        """Allocate kv_pool + workspace with torch (1024-byte aligned) and create the handle."""
        import torch
        pool_bytes, ws_bytes = query_sizes(cfg)
        dt = torch.bfloat16 if cfg.kv_dtype == DELTA_BF16 else torch.float32
        shape = (cfg.num_layers, cfg.phys_pages, cfg.num_kv_heads, 2, cfg.page_size, cfg.head_dim)
        # the caching allocator guarantees 512-byte alignment only: over-allocate and align the
        # pool to the 1024 bytes its TMA descriptor (128-byte swizzle) needs
        raw = torch.zeros(pool_bytes + 1024, dtype=torch.uint8, device=device)
        off = (-raw.data_ptr()) % 1024
        kv_pool = raw[off: off + pool_bytes].view(dt).view(shape)
        assert kv_pool.data_ptr() % 1024 == 0
        ws = torch.zeros(ws_bytes, dtype=torch.uint8, device=device)
        bt = block_table.to(device=device, dtype=torch.int32).contiguous()
        return cls(cfg, kv_pool, bt, ws)

    # ------------------------------------------------------------------ argument checks
    def _arg(self, t, kind: str, shape, name: str, host: bool = False):
        """Marshalling checks only (no arithmetic): dtype, contiguity, device and shape of a tensor
        argument before its raw pointer crosses the C ABI (which cannot check them)."""
        import torch
        dt = {"kv": torch.bfloat16 if self.cfg.kv_dtype == DELTA_BF16 else torch.float32,
              "f32": torch.float32, "i32": torch.int32}[kind]
        if t.dtype != dt:
            raise DeltaError(2, f"{name}: dtype {t.dtype}, expected {dt}")
        if not t.is_contiguous():
            raise DeltaError(2, f"{name}: must be contiguous")
        if host:
            if t.is_cuda:
                raise DeltaError(2, f"{name}: must be a host tensor")
        elif not t.is_cuda or t.device != self.kv_pool.device:
            raise DeltaError(2, f"{name}: must live on {self.kv_pool.device}")
        if len(t.shape) != len(shape) or any(e is not None and a != e for a, e in zip(t.shape, shape)):
            raise DeltaError(2, f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)} (None = any)")
        return t.data_ptr()

    def _opt(self, t, kind, shape, name, host=False):
        return None if t is None else self._arg(t, kind, shape, name, host)

    # ------------------------------------------------------------------ calls
    def set_seq_lens(self, lens, layer: int = -1, stream=None):
        arr = (ctypes.c_int32 * len(lens))(*[int(x) for x in lens])
        _check(self.lib.delta_set_seq_lens(self.h, layer, len(lens), arr, _stream(stream)), self.h)

    def append_kv(self, layer: int, k_new, v_new, stream=None):
        c = self.cfg
        batch, ntok = k_new.shape[0], k_new.shape[1]
        kp = self._arg(k_new, "kv", (batch, ntok, c.num_kv_heads, c.head_dim), "k_new")
        vp_ = self._arg(v_new, "kv", (batch, ntok, c.num_kv_heads, c.head_dim), "v_new")
        _check(self.lib.delta_append_kv(self.h, layer, batch, ntok, kp, vp_, _stream(stream)), self.h)

    def decode_layer(self, layer: int, q, out, lse=None, stream=None):
        c = self.cfg
        b = q.shape[0]
        qp = self._arg(q, "kv", (b, c.num_q_heads, c.head_dim), "q")
        op = self._arg(out, "f32", (b, c.num_q_heads, c.head_dim), "out")
        lp = self._opt(lse, "f32", (b, c.num_q_heads), "lse")
        _check(self.lib.delta_decode_layer(self.h, layer, b, qp, op, lp, _stream(stream)), self.h)

    def append_decode_layer(self, layer: int, k_new, v_new, q, out, lse=None, stream=None):
        c = self.cfg
        b = q.shape[0]
        kp = self._arg(k_new, "kv", (b, c.num_kv_heads, c.head_dim), "k_new")
        vp_ = self._arg(v_new, "kv", (b, c.num_kv_heads, c.head_dim), "v_new")
        qp = self._arg(q, "kv", (b, c.num_q_heads, c.head_dim), "q")
        op = self._arg(out, "f32", (b, c.num_q_heads, c.head_dim), "out")
        lp = self._opt(lse, "f32", (b, c.num_q_heads), "lse")
        _check(self.lib.delta_append_decode_layer(self.h, layer, b, kp, vp_, qp, op, lp, _stream(stream)), self.h)

    def select(self, layer: int, batch: int, keys_override=None, idx_out=None, count_out=None, stream=None):
        cap = self.plan_capacity
        kp = self._opt(keys_override, "f32", (batch, None), "keys_override")
        ip = self._opt(idx_out, "i32", (batch, cap), "idx_out")
        cp = self._opt(count_out, "i32", (batch,), "count_out")
        _check(self.lib.delta_select(self.h, layer, batch, kp, ip, cp, _stream(stream)), self.h)

    def quest_build_reps(self, layer: int = -1, batch: int | None = None, stream=None):
        _check(self.lib.delta_quest_build_reps(self.h, layer, batch or self.cfg.max_batch, _stream(stream)), self.h)

    def raas_reset(self, layer: int = -1, batch: int | None = None, stream=None):
        _check(self.lib.delta_raas_reset(self.h, layer, batch or self.cfg.max_batch, _stream(stream)), self.h)

    def copy_plan(self, layer: int, batch: int, idx_out, count_out, stream=None):
        _check(self.lib.delta_copy_plan(self.h, layer, batch, _ptr(idx_out), _ptr(count_out), _stream(stream)),
               self.h)

    def attention_recall(self, layer: int, q, recall_out, stream=None):
        """Eq.9 recall [batch][m] of the plan `layer` attended this step (diagnostic)."""
        _check(self.lib.delta_attention_recall(self.h, layer, q.shape[0], q.data_ptr(), recall_out.data_ptr(),
                                               _stream(stream)), self.h)

    def prefill(self, layer: int, q, k_new, v_new, out, lse=None, stream=None):
        """Chunked prefill: append q.shape[1] tokens and attend causally (q [B][ntok][m][d])."""
        c = self.cfg
        b, n = q.shape[0], q.shape[1]
        qp = self._arg(q, "kv", (b, n, c.num_q_heads, c.head_dim), "q")
        kp = self._arg(k_new, "kv", (b, n, c.num_kv_heads, c.head_dim), "k_new")
        vp_ = self._arg(v_new, "kv", (b, n, c.num_kv_heads, c.head_dim), "v_new")
        op = self._arg(out, "f32", (b, n, c.num_q_heads, c.head_dim), "out")
        lp = self._opt(lse, "f32", (b, n, c.num_q_heads), "lse")
        _check(self.lib.delta_prefill(self.h, layer, b, n, qp, kp, vp_, op, lp, _stream(stream)), self.h)

    def workspace_region(self, which: int):
        """(device pointer, bytes) of a workspace region (0 unit keys, 1 Quest reps)."""
        ptr, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check(self.lib.delta_workspace_region(self.h, which, ctypes.byref(ptr), ctypes.byref(n)), self.h)
        return ptr.value, n.value

    def decode_step(self, q_all, k_all, v_all, out_all, lse_all=None, stream=None):
        c = self.cfg
        L, b = c.num_layers, q_all.shape[1]
        qp = self._arg(q_all, "kv", (L, b, c.num_q_heads, c.head_dim), "q_all")
        kp = self._arg(k_all, "kv", (L, b, c.num_kv_heads, c.head_dim), "k_all")
        vp_ = self._arg(v_all, "kv", (L, b, c.num_kv_heads, c.head_dim), "v_all")
        op = self._arg(out_all, "f32", (L, b, c.num_q_heads, c.head_dim), "out_all")
        lp = self._opt(lse_all, "f32", (L, b, c.num_q_heads), "lse_all")
        _check(self.lib.delta_decode_step(self.h, b, qp, kp, vp_, op, lp, _stream(stream)), self.h)

    def decode_step_host(self, q_host, k_host, v_host, out_host, stream=None):
        c = self.cfg
        L, b = c.num_layers, q_host.shape[1]
        qp = self._arg(q_host, "kv", (L, b, c.num_q_heads, c.head_dim), "q_host", host=True)
        kp = self._arg(k_host, "kv", (L, b, c.num_kv_heads, c.head_dim), "k_host", host=True)
        vp_ = self._arg(v_host, "kv", (L, b, c.num_kv_heads, c.head_dim), "v_host", host=True)
        op = self._arg(out_host, "f32", (L, b, c.num_q_heads, c.head_dim), "out_host", host=True)
        _check(self.lib.delta_decode_step_host(self.h, b, qp, kp, vp_, op, _stream(stream)), self.h)

    def exchange_buffers(self, which: int):
        """(send_ptr, recv_ptr, block_bytes) of the external exchange (0: attention, 1: candidates)."""
        s_, r_, n_ = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_size_t()
        _check(self.lib.delta_shard_exchange_buffers(self.h, which, ctypes.byref(s_), ctypes.byref(r_),
                                                     ctypes.byref(n_)), self.h)
        return s_.value, r_.value, n_.value

    def shard_merge(self, layer: int, out, lse=None, stream=None):
        _check(self.lib.delta_shard_merge(self.h, layer, out.shape[0], out.data_ptr(), _ptr(lse), _stream(stream)),
               self.h)

    def shard_select_merge(self, layer: int, batch: int, idx_out=None, count_out=None, stream=None):
        _check(self.lib.delta_shard_select_merge(self.h, layer, batch, _ptr(idx_out), _ptr(count_out),
                                                 _stream(stream)), self.h)

    def get_error(self, stream=None) -> int:
        v = ctypes.c_int()
        _check(self.lib.delta_get_error(self.h, _stream(stream), ctypes.byref(v)), self.h)
        return v.value

    def role(self, layer: int) -> int:
        return self.lib.delta_layer_role(self.h, layer)

    def governing(self, layer: int) -> int:
        return self.lib.delta_governing_layer(self.h, layer)

    @property
    def plan_capacity(self) -> int:
        return self.lib.delta_plan_capacity(self.h)

    @property
    def kernels_launched(self) -> int:
        return int(self.lib.delta_kernels_launched(self.h))

    def kernel_name(self, layer: int, batch: int) -> str:
        """The attention kernel variant a decode of `layer` at `batch` launches."""
        return self.lib.delta_layer_kernel_name(self.h, layer, batch).decode()

    @property
    def graph_captures(self) -> int:
        return int(self.lib.delta_graph_captures(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.delta_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
