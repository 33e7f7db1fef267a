"""Python handle on the sm_100a device half of the C ABI (include/lkv.h).

torch is used only as plumbing: device buffers for K/V/q/out and stream
wrappers. All data movement and attention run in liblkv.so's kernels and
copy-engine streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _abi
from .layersim import KvManager, ModelSpec

DTYPE_BF16, DTYPE_F32 = 0, 1


@dataclass
class DeviceConfig:
    device: int = 0
    tp_rank: int = 0
    tp_size: int = 1
    pipeline_depth: int = 2
    gpu_slots: int = 0
    host_slots: int = 0
    arena_slots: int = 0
    max_requests: int = 64
    max_blocks: int = 4096
    max_batch: int = 64
    staging_chunks: int = 4
    chunk_bytes: int = 16 << 20
    pinned_frames: int = 0  # > 0: tiered host memory (pageable homes + this many pinned frames)

    def c(self):
        return _abi.DeviceConfig(self.device, self.tp_rank, self.tp_size, self.pipeline_depth, self.gpu_slots,
                                 self.host_slots, self.arena_slots, self.max_requests, self.max_blocks,
                                 self.max_batch, self.staging_chunks, self.chunk_bytes, self.pinned_frames)


def _ptr(t) -> int:
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: CUDA's legacy default stream, torch's default stream


def _stream(stream):
    """Caller's stream handle: the given torch stream, else torch's current
    stream on the current device (so tensors produced there are ordered).
    torch's default stream is CUDA's legacy stream 0; it is passed as
    cudaStreamLegacy, because a NULL handle means "the device's compute
    stream" in the C ABI — passing 0 would drop the ordering with the
    caller's tensors (the non-blocking compute stream does not synchronise
    with stream 0), and the caching allocator could recycle an input (e.g.
    a freed q) before the kernel reads it."""
    if stream is None:
        try:
            import torch
            stream = torch.cuda.current_stream()
        except Exception:
            return None
    return C.c_void_p(stream.cuda_stream or _CUDA_STREAM_LEGACY)


def _device_view(ptr: int, shape, dtype, device: int):
    """A torch tensor aliasing device memory owned by liblkv (no copy)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<i2", "data": (ptr, False), "version": 3,
                                    "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_Arr(), device=torch.device("cuda", device)).view(dtype)


def numa_node(cuda_device: int) -> int:
    """NUMA node of a CUDA device (include/lkv.h lkv_device_numa_node); -1
    when unknown or single-node."""
    n = C.c_int32()
    _abi.product_lib().call("lkv_device_numa_node", cuda_device, C.byref(n))
    return n.value


def bind_to_numa_node(cuda_device: int) -> dict:
    """Pin this process's threads to the CPUs of the GPU's NUMA node, so host
    buffers it allocates (first touch) and the copy threads sit next to the
    GPU's PCIe link. No-op on single-node hosts."""
    import os
    node = numa_node(cuda_device)
    nodes = [d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")] \
        if os.path.isdir("/sys/devices/system/node") else []
    out = {"numa_node": node, "numa_nodes": len(nodes), "cpus": None}
    if node < 0 or len(nodes) < 2:
        return out
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            cpus = set()
            for part in f.read().strip().split(","):
                lo, _, hi = part.partition("-")
                cpus.update(range(int(lo), int(hi or lo) + 1))
        os.sched_setaffinity(0, cpus)
        out["cpus"] = len(cpus)
    except OSError:
        pass
    return out


class Device:
    """One GPU's KV-head shard of the LayerKV data path, bound to a KvManager."""

    def __init__(self, kv: KvManager, model: ModelSpec, tokens_per_block: int, cfg: DeviceConfig, lib=None):
        self._lib = lib or _abi.product_lib()
        if not self._lib.has_device:
            raise RuntimeError("library has no device half")
        self.kv = kv  # keep the manager alive while bound
        self.model = model
        self.cfg = cfg
        h = C.c_void_p()
        self._lib.call("lkv_device_create", C.byref(model.c()), tokens_per_block, C.byref(cfg.c()), C.byref(h))
        self.handle = h
        self._lib.call("lkv_device_bind", h, kv.handle)
        info = _abi.DeviceInfo()
        self._lib.call("lkv_device_get_info", h, C.byref(info))
        self.info = info
        self.slot_bytes = info.slot_bytes
        self.kv_heads_local = info.kv_heads_local
        self.q_heads_local = info.q_heads_local
        self.head_dim = info.head_dim
        self.tokens_per_block = info.tokens_per_block
        self.head0 = cfg.tp_rank * info.kv_heads_local

    def close(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.dll.lkv_device_destroy(h)
            self.handle = None

    def __del__(self):
        self.close()

    # ------------------------------------------------------------- streams
    def torch_stream(self, which: str = "compute"):
        import torch
        ptr = {"compute": self.info.compute_stream, "d2h": self.info.d2h_stream, "h2d": self.info.h2d_stream}[which]
        return torch.cuda.ExternalStream(ptr, device=torch.device("cuda", self.cfg.device))

    def synchronize(self):
        self._lib.call("lkv_device_synchronize", self.handle)

    def set_timing(self, on: bool):
        self._lib.call("lkv_device_set_timing", self.handle, int(on))

    # ------------------------------------------------------------- prefill
    def prefill_layer(self, request_id: int, layer: int, k, v, tokens: int, stream=None):
        self._lib.call("lkv_prefill_layer", self.handle, request_id, layer, _ptr(k), _ptr(v), tokens,
                       _stream(stream))

    def prefill_attention(self, q, k, v, out, tokens: int, scale: float, out_dtype: int = DTYPE_BF16, stream=None):
        """Causal GQA attention of one prefill layer on the tensor cores:
        q/out [tokens][q_heads_local][d], k/v [tokens][kv_heads_local][d] (bf16; out bf16 or fp32)."""
        self._lib.call("lkv_prefill_attention", self.handle, _ptr(q), _ptr(k), _ptr(v), _ptr(out), tokens, scale,
                       out_dtype, _stream(stream))

    def prefill_offload_done(self, request_id: int) -> bool:
        out = C.c_int32()
        self._lib.call("lkv_device_prefill_offload_done", self.handle, request_id, C.byref(out))
        return bool(out.value)

    def job_done(self, job_id: int) -> bool:
        out = C.c_int32()
        self._lib.call("lkv_device_job_done", self.handle, job_id, C.byref(out))
        return bool(out.value)

    # ------------------------------------------------------------- decode
    def decode_begin(self, request_ids):
        arr = (C.c_int64 * max(1, len(request_ids)))(*request_ids)
        self._lib.call("lkv_decode_begin", self.handle, arr, len(request_ids))

    def decode_begin_append(self, request_ids):
        """Serving decode: this iteration appends one token per member (f2)."""
        arr = (C.c_int64 * max(1, len(request_ids)))(*request_ids)
        self._lib.call("lkv_decode_begin_append", self.handle, arr, len(request_ids))

    def decode_append_layer(self, layer: int, k_new, v_new, stream=None):
        self._lib.call("lkv_decode_append_layer", self.handle, layer, _ptr(k_new), _ptr(v_new), _stream(stream))

    def decode_layer(self, layer: int, q, out, scale: float, out_dtype: int = DTYPE_BF16, stream=None):
        """Paged attention of one layer; ordered after `stream`'s queued work
        (default: torch's current stream), which in turn waits for `out`."""
        self._lib.call("lkv_decode_layer", self.handle, layer, _ptr(q), _ptr(out), scale, out_dtype, _stream(stream))

    def decode_end(self):
        self._lib.call("lkv_decode_end", self.handle)

    # ------------------------------------------------------------- fused all-gather
    def gather_ipc_handle(self) -> bytes:
        """This rank's gather-buffer IPC handle, to exchange out of band."""
        buf = C.create_string_buffer(_abi.IPC_HANDLE_BYTES)
        self._lib.call("lkv_device_gather_ipc_handle", self.handle, buf)
        return buf.raw

    def gather_connect_ipc(self, handles):
        """Connect with every rank's handle (rank order, own included)."""
        blob = b"".join(handles)
        if len(blob) != _abi.IPC_HANDLE_BYTES * len(handles):
            raise ValueError("gather handles must be 64 bytes each")
        self._lib.call("lkv_device_gather_connect_ipc", self.handle, blob, len(handles))

    def gather_buffer(self) -> int:
        base, n = C.c_void_p(), C.c_uint64()
        self._lib.call("lkv_device_gather_buffer", self.handle, C.byref(base), C.byref(n))
        return base.value

    def gather_connect(self, bases):
        """Same-process ranks: connect with each rank's gather_buffer() pointer."""
        arr = (C.c_void_p * len(bases))(*bases)
        self._lib.call("lkv_device_gather_connect", self.handle, arr, len(bases))

    def placement(self) -> dict:
        """Where this rank's resources sit: the NUMA node its pinned host pool
        was bound to (-1: none / single node) and how many gather peers on
        other GPUs it reaches over P2P (after gather_connect*)."""
        info = _abi.DeviceInfo()
        self._lib.call("lkv_device_get_info", self.handle, C.byref(info))
        return {"numa_node": info.numa_node, "gather_peers_p2p": info.gather_peers}

    def gather_wait(self, layer: int, stream=None):
        """Enqueue on `stream` a wait for every rank's rows of `layer`."""
        self._lib.call("lkv_decode_gather_wait", self.handle, layer, _stream(stream))

    def gathered(self, layer: int):
        """torch view [max_batch, q_heads_local * tp_size, head_dim] bf16 of
        layer's gathered rows (valid on a stream after gather_wait)."""
        import torch
        p = C.c_void_p()
        self._lib.call("lkv_decode_gathered", self.handle, layer, C.byref(p))
        shape = (self.cfg.max_batch, self.q_heads_local * self.cfg.tp_size, self.head_dim)
        return _device_view(p.value, shape, torch.bfloat16, self.cfg.device)

    def decode_stats(self) -> _abi.DecodeStats:
        s = _abi.DecodeStats()
        self._lib.call("lkv_decode_last_stats", self.handle, C.byref(s))
        return s

    def offload_stats(self, reset: bool = False) -> _abi.OffloadStats:
        s = _abi.OffloadStats()
        self._lib.call("lkv_offload_last_stats", self.handle, C.byref(s), int(reset))
        return s

    # ------------------------------------------------------------- synthetic data
    def fill_kv(self, k, v, tokens: int, token0: int, layer: int, seed: int, stream=None):
        s = None if stream is None else C.c_void_p(stream.cuda_stream)
        self._lib.call("lkv_fill_kv", self.handle, _ptr(k), _ptr(v), tokens, token0, layer, seed, s)

    def verify_request(self, request_id: int, n_tokens: int, seed: int) -> int:
        out = C.c_int64()
        self._lib.call("lkv_verify_request", self.handle, request_id, n_tokens, seed, C.byref(out))
        return out.value

    def fill_request(self, request_id: int, n_tokens: int, seed: int):
        self._lib.call("lkv_fill_request", self.handle, request_id, n_tokens, seed)

    # ------------------------------------------------------------- raw views (tests)
    def read_host_slot(self, slot: int) -> bytes:
        """Bytes of one CPU slot, wherever they live (pinned frame, or its
        pageable home in tiered mode)."""
        buf = C.create_string_buffer(self.slot_bytes)
        self._lib.call("lkv_device_read_host_slot", self.handle, slot, buf)
        return buf.raw

    def free_stack(self, gpu: bool = True):
        """The device (HBM) mirror of the manager's free list, in
        KvManager.free_stack's form (bottom to top)."""
        n = C.c_int64()
        which = 0 if gpu else 1
        self._lib.call("lkv_device_free_stack", self.handle, which, None, 0, C.byref(n))
        out = (C.c_uint32 * max(1, n.value))()
        self._lib.call("lkv_device_free_stack", self.handle, which, out, n.value, C.byref(n))
        return list(out)[:n.value]

    def host_tier_stats(self) -> _abi.HostTierStats:
        s = _abi.HostTierStats()
        self._lib.call("lkv_device_host_tier_stats", self.handle, C.byref(s))
        return s
