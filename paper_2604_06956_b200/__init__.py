"""NestPipe (arXiv 2604.06956) sharded-embedding hot path on B200.

Thin Python binding over libnest.so (include/nest.h): every step of the path
runs in the library's sm_100a kernels and NCCL calls; this module only
allocates device memory with torch, marshals pointers and streams, and raises
on error.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

from . import _lib as L
from ._lib import NestError  # noqa: F401

__all__ = ["NestContext", "NestError", "unique_ids", "connect_windows"]


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(s) -> Optional[int]:
    if s is None:
        import torch
        s = torch.cuda.current_stream()
    return s.cuda_stream


def unique_ids() -> bytes:
    """Two NCCL unique ids (main + aux communicator), 256 bytes; call on rank 0."""
    lib = L.load()
    buf = C.create_string_buffer(256)
    L.check(lib.nest_get_unique_id(C.byref(buf, 0)))
    L.check(lib.nest_get_unique_id(C.byref(buf, 128)))
    return buf.raw


class NestContext:
    """One rank's context: shard + workspace (torch-allocated) + libnest ctx."""

    def __init__(self, table_rows: Sequence[int], dim: int, *, world: int = 1, rank: int = 0,
                 pooling: str = "sum", num_features: Optional[int] = None, max_keys: int,
                 max_batch: int, max_micro_batches: int = 1, max_recv_keys: int = 0,
                 max_mb_rows: int = 0, max_owner_mb_rows: int = 0, seed: int = 0,
                 init_mode: str = "uniform", tower_layers: int = 0, tower_hidden: int = 1024,
                 optimizer: str = "sgd", adagrad_eps: float = 1e-8, table_location: str = "hbm",
                 tower_train: bool = False, tower_lr: float = 1e-3,
                 nccl_uids: Optional[bytes] = None, device=None, init_tables: bool = True):
        import torch
        self.lib = L.load()
        self.torch = torch
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._rows = (C.c_int64 * len(table_rows))(*[int(r) for r in table_rows])
        self.cfg = L.Config(
            world=world, rank=rank, num_tables=len(table_rows), dim=dim, table_rows=self._rows,
            pooling={"sum": L.POOL_SUM, "none": L.POOL_NONE}[pooling],
            num_features=num_features if num_features is not None else len(table_rows),
            max_keys=max_keys, max_batch=max_batch, max_micro_batches=max_micro_batches,
            max_recv_keys=max_recv_keys, max_owner_keys=0, max_mb_rows=max_mb_rows,
            max_owner_mb_rows=max_owner_mb_rows, seed=seed,
            init_mode={"uniform": L.INIT_UNIFORM, "dyadic": L.INIT_DYADIC, "zero": L.INIT_ZERO}[init_mode],
            tower_layers=tower_layers, tower_hidden=tower_hidden,
            optimizer={"sgd": L.OPT_SGD, "rowwise_adagrad": L.OPT_ROWWISE_ADAGRAD}[optimizer],
            adagrad_eps=adagrad_eps,
            table_location={"hbm": L.TABLE_HBM, "host": L.TABLE_HOST}[table_location],
            tower_train=1 if tower_train else 0, tower_lr=tower_lr)
        self.table_location = table_location
        self.optimizer = optimizer
        self.world, self.rank, self.dim = world, rank, dim
        self.F = self.cfg.num_features
        tb, wb = C.c_size_t(), C.c_size_t()
        L.check(self.lib.nest_workspace_bytes(C.byref(self.cfg), C.byref(tb), C.byref(wb)))
        self.table_bytes, self.work_bytes = tb.value, wb.value
        self.shard_rows = self.lib.nest_shard_rows(C.byref(self.cfg))
        with torch.cuda.device(self.device):
            if table_location == "host":
                # host-DRAM tier (NEXT-3): pinned host memory, reached by the
                # kernels over PCIe through its UVA device alias
                self.table_mem = torch.empty(self.table_bytes, dtype=torch.uint8, pin_memory=True)
            else:
                self.table_mem = torch.empty(self.table_bytes, dtype=torch.uint8, device=self.device)
            self.work_mem = torch.empty(self.work_bytes, dtype=torch.uint8, device=self.device)
            self.shard = self.table_mem.view(torch.float32)[: self.shard_rows * dim].view(self.shard_rows, dim)
            ctx = C.c_void_p()
            uid = None
            if world > 1 and nccl_uids is not None:
                if len(nccl_uids) != 256:
                    raise ValueError("nccl_uids must be the 256 bytes of unique_ids() from rank 0")
                uid = C.create_string_buffer(nccl_uids, 256)
            # world > 1 without nccl_uids: no NCCL, exchanges over the peer
            # windows; connect them with window_export / window_connect
            st = torch.cuda.current_stream(self.device)
            L.check(self.lib.nest_create(C.byref(self.cfg), uid, _ptr(self.table_mem), _ptr(self.work_mem),
                                         st.cuda_stream, C.byref(ctx)))
            self.ctx = ctx
            if init_tables:
                self.init_tables(st)

    # -- NCCL-free mode: exchange-window rendezvous -----------------------------
    def window_export(self) -> bytes:
        """This rank's window record (nest_window_export), to be moved to every
        rank by the caller (torch.distributed.all_gather_object, or in-process)."""
        rec = L.WindowRec()
        self._check(self.lib.nest_window_export(self.ctx, C.byref(rec)))
        return bytes(rec)

    def window_connect(self, recs: Sequence[bytes]) -> None:
        """Map every rank's window (records in rank order; nest_window_connect)."""
        arr = (L.WindowRec * len(recs))()
        for i, r in enumerate(recs):
            C.memmove(C.byref(arr, i * C.sizeof(L.WindowRec)), r, C.sizeof(L.WindowRec))
        self._check(self.lib.nest_window_connect(self.ctx, arr))

    def check_guards(self, stream=None) -> int:
        """Checked mode (NEST_GUARD=1 at creation): number of overwritten guard
        words after the workspace buffers (nest_check_guards; 0 = intact)."""
        n = C.c_int64()
        self._check(self.lib.nest_check_guards(self.ctx, _stream(stream), C.byref(n)))
        return int(n.value)

    # -- lifecycle -----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "ctx", None):
            self.lib.nest_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, code: int) -> None:
        L.check(code, self.ctx)

    # -- calls (1:1 with include/nest.h) -------------------------------------
    def init_tables(self, stream=None) -> None:
        self._check(self.lib.nest_init_tables(self.ctx, _stream(stream)))

    def fwp_schedule(self, keys, bag_offsets, B: int, N: int, mode: str = "sequential", stream=None):
        torch = self.torch
        perm = torch.empty(B, dtype=torch.int32, device=self.device)
        mbo = torch.empty(N + 1, dtype=torch.int32, device=self.device)
        m = {"sequential": L.SCHED_SEQUENTIAL, "clustered": L.SCHED_CLUSTERED}[mode]
        nnz = 0 if keys is None else int(keys.numel())
        self._check(self.lib.nest_fwp_schedule(self.ctx, _ptr(keys), _ptr(bag_offsets), nnz, B, N, m,
                                               _ptr(perm), _ptr(mbo), _stream(stream)))
        return perm, mbo

    def route(self, slot: int, keys, bag_offsets, B: int, perm=None, mb_offsets=None, N: int = 1,
              stream=None) -> None:
        self._check(self.lib.nest_route(self.ctx, slot, _ptr(keys), _ptr(bag_offsets), int(keys.numel()),
                                        B, _ptr(perm), _ptr(mb_offsets), N, _stream(stream)))

    def route_begin(self, slot: int, keys, bag_offsets, B: int, perm=None, mb_offsets=None, N: int = 1,
                    stream=None) -> None:
        """First half of route (no host sync): nest_route_begin."""
        self._check(self.lib.nest_route_begin(self.ctx, slot, _ptr(keys), _ptr(bag_offsets), int(keys.numel()),
                                              B, _ptr(perm), _ptr(mb_offsets), N, _stream(stream)))

    def route_end(self, slot: int) -> None:
        """Second half of route (the host sync on the counts): nest_route_end."""
        self._check(self.lib.nest_route_end(self.ctx, slot))

    def dbp_refresh(self, active: int, prefetch: int, stream=None) -> None:
        self._check(self.lib.nest_dbp_refresh(self.ctx, active, prefetch, _stream(stream)))

    def lookup_prefetch(self, slot: int, mb: int, compute=None, comm=None) -> None:
        self._check(self.lib.nest_lookup_prefetch(self.ctx, slot, mb, _stream(compute),
                                                  _stream(comm if comm is not None else compute)))

    def lookup_fwd(self, slot: int, mb: int, out, compute=None, comm=None) -> None:
        """Pool micro-batch mb into `out` (fp32, or bf16 -> nest_lookup_fwd_bf16)."""
        fn = self.lib.nest_lookup_fwd_bf16 if str(out.dtype) == "torch.bfloat16" else self.lib.nest_lookup_fwd
        self._check(fn(self.ctx, slot, mb, _ptr(out), _stream(compute),
                       _stream(comm if comm is not None else compute)))

    def grad_bwd_update(self, slot: int, mb: int, dout, lr_over_B: float, compute=None, comm=None) -> None:
        self._check(self.lib.nest_grad_bwd_update(self.ctx, slot, mb, _ptr(dout), float(lr_over_B),
                                                  _stream(compute),
                                                  _stream(comm if comm is not None else compute)))

    def grad_bwd_update_adagrad(self, slot: int, mb: int, dout, grad_scale: float, lr: float, compute=None,
                                comm=None) -> None:
        self._check(self.lib.nest_grad_bwd_update_adagrad(self.ctx, slot, mb, _ptr(dout), float(grad_scale),
                                                          float(lr), _stream(compute),
                                                          _stream(comm if comm is not None else compute)))

    def tower_fwd_bwd(self, pooled, dout, stream=None) -> None:
        """Stand-in tower on fp32 or bf16 pooled rows (-> nest_tower_fwd_bwd_bf16)."""
        fn = self.lib.nest_tower_fwd_bwd_bf16 if str(pooled.dtype) == "torch.bfloat16" else self.lib.nest_tower_fwd_bwd
        self._check(fn(self.ctx, _ptr(pooled), int(pooled.shape[0]), _ptr(dout), _stream(stream)))

    def set_zero_copy(self, on: bool) -> None:
        """Zero-copy retrieval for W=1 / N=1 / HBM batches routed from now on
        (nest_set_zero_copy)."""
        self._check(self.lib.nest_set_zero_copy(self.ctx, 1 if on else 0))

    def set_streams(self, sort_stream=None, tower_dw_stream=None) -> None:
        """The library's internal streams -> the caller's (nest_set_streams)."""
        self._check(self.lib.nest_set_streams(self.ctx, sort_stream.cuda_stream if sort_stream is not None else None,
                                              tower_dw_stream.cuda_stream if tower_dw_stream is not None else None))

    def tower_step(self, stream=None) -> None:
        """Trained tower: AllReduce + SGD of the batch's accumulated dW, once
        after its last micro-batch (nest_tower_step; no-op for the fixed tower)."""
        self._check(self.lib.nest_tower_step(self.ctx, _stream(stream)))

    def tower_read(self, what: str, layer: int = 0, stream=None):
        """The tower's layer weights [H, in_l] or its fixed top gradient
        [max_batch, H] as an fp32 device tensor (nest_tower_read)."""
        torch = self.torch
        H, in0 = self.cfg.tower_hidden, self.F * self.dim
        shape = ((H, in0 if layer == 0 else H) if what == "weights" else (self.cfg.max_batch, H))
        out = torch.empty(shape, dtype=torch.float32, device=self.device)
        self._check(self.lib.nest_tower_read(self.ctx, {"weights": 0, "top_grad": 1}[what], layer, _ptr(out),
                                             _stream(stream)))
        return out

    def join(self, stream=None) -> None:
        """`stream` waits for the library's internal streams (nest_join)."""
        self._check(self.lib.nest_join(self.ctx, _stream(stream)))

    def slot_info(self, slot: int) -> L.SlotInfo:
        info = L.SlotInfo()
        self._check(self.lib.nest_slot_info(self.ctx, slot, C.byref(info)))
        return info

    def out_rows(self, slot: int, mb: int) -> int:
        return int(self.slot_info(slot).mb_out_rows[mb])

    def read_rows(self, keys, stream=None):
        torch = self.torch
        out = torch.empty((int(keys.numel()), self.dim), dtype=torch.float32, device=self.device)
        self._check(self.lib.nest_read_rows(self.ctx, _ptr(keys), int(keys.numel()), _ptr(out),
                                            _stream(stream)))
        return out

    def read_state(self, keys, stream=None):
        """Row-wise AdaGrad accumulators of owned keys (nest_read_state)."""
        torch = self.torch
        out = torch.empty(int(keys.numel()), dtype=torch.float32, device=self.device)
        self._check(self.lib.nest_read_state(self.ctx, _ptr(keys), int(keys.numel()), _ptr(out), _stream(stream)))
        return out

    def profile_enable(self, on: bool = True) -> None:
        self._check(self.lib.nest_profile_enable(self.ctx, 1 if on else 0))

    def profile_read(self) -> dict:
        stages = (L.ProfileStage * L.PROFILE_STAGES)()
        summ = L.ProfileSummary()
        self._check(self.lib.nest_profile_read(self.ctx, stages, C.byref(summ)))
        out = {"stages": {}, "summary": {k: getattr(summ, k) for k, _ in L.ProfileSummary._fields_}}
        for s in stages:
            out["stages"][s.name.decode()] = {"stream": s.stream, "records": s.records,
                                              "launches": s.launches, "ms": s.ms, "bytes": s.bytes,
                                              "units": s.units, "hbm_bytes": s.hbm_bytes}
        return out

    def profile_records(self) -> list:
        """The trace's raw stage intervals: [(stage name, stream kind, t0 ms, t1 ms)]."""
        n = C.c_int64()
        self._check(self.lib.nest_profile_records(self.ctx, None, 0, C.byref(n)))
        recs = (L.ProfileRecord * max(1, n.value))()
        self._check(self.lib.nest_profile_records(self.ctx, recs, n.value, C.byref(n)))
        names = list(self.profile_read()["stages"].keys())
        kinds = {0: "compute", 1: "comm", 2: "aux"}
        return [(names[r.stage], kinds.get(r.stream, str(r.stream)), r.t0_ms, r.t1_ms) for r in recs[:n.value]]

    def route_view(self, slot: int) -> dict:
        """Copies of a slot's routing results (host numpy) for parity checks."""
        torch = self.torch
        import numpy as np
        v = L.RouteView()
        self._check(self.lib.nest_route_view(self.ctx, slot, C.byref(v)))
        info = self.slot_info(slot)
        torch.cuda.synchronize(self.device)
        N, W = info.num_micro_batches, self.world
        Nc = self.cfg.max_micro_batches + 2
        K = int(self.cfg.max_keys)

        def fetch(addr, n, dtype):
            n = int(n)
            if n == 0 or not addr:
                return np.zeros(0, dtype=dtype)
            out = np.empty(n, dtype=dtype)
            _memcpy_d2h(out.ctypes.data, addr, out.nbytes)
            return out

        U = int(info.uniq)
        n_owner = int(fetch(v.n_owner, 1, np.int32)[0])
        out = {
            "uniq": fetch(v.uniq, U, np.int64),
            "inverse": fetch(v.inverse, info.nnz, np.int32),
            "mask": fetch(v.mask, U, np.uint32),
            "pos": np.stack([fetch(v.pos + 4 * i * (K + 1), U, np.int32) for i in range(N)]) if N else None,
            "send_counts": fetch(v.send_counts, W * Nc, np.int32).reshape(W, Nc),
            "all_counts": fetch(v.all_counts, W * W * Nc, np.int32).reshape(W, W, Nc),
            "owner_rows": fetch(v.owner_rows, n_owner, np.int32),
            "n_owner": n_owner,
            "buffer": fetch(v.buffer, n_owner * self.dim, np.float32).reshape(n_owner, self.dim),
            "info": info,
        }
        if W > 1:
            out["recv_keys"] = fetch(v.recv_keys, info.recv, np.int64)
            out["owner_inv"] = fetch(v.owner_inv, info.recv, np.int32)
        return out


_cudart = None


def _memcpy_d2h(dst: int, src: int, nbytes: int) -> None:
    """Synchronous device->host copy through the CUDA runtime torch loaded."""
    global _cudart
    if _cudart is None:
        import os
        import torch  # noqa: F401  (loads libcudart.so.12 into the process)
        try:
            _cudart = C.CDLL("libcudart.so.12")
        except OSError:
            import nvidia.cuda_runtime as cr
            _cudart = C.CDLL(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so.12"))
        _cudart.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
        _cudart.cudaMemcpy.restype = C.c_int
    rc = _cudart.cudaMemcpy(dst, src, nbytes, 2)  # cudaMemcpyDeviceToHost
    if rc != 0:
        raise NestError(2, f"cudaMemcpy failed ({rc})")


def connect_windows(contexts) -> None:
    """Connect the ranks of one process (e.g. several ranks on one device,
    each driven by its own thread): every context maps every other's window."""
    recs = [c.window_export() for c in contexts]
    for c in contexts:
        c.window_connect(recs)
