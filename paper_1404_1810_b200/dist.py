"""Multi-GPU plumbing (one process per GPU, torch.distributed).

Batched AM-QFT workloads shard by rows with no data-path collective: rank r
owns rows [start, start + count) of the global batch, runs its own plan on
its own device, and only the timing (max over ranks) and optional result
gathering use the process group.

A single huge transform (BASELINE config 5, N = 2^30 over P GPUs; SURVEY
8(e)) runs as a distributed four-step with exactly one exchange step:
`DistFourStep` below.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

import ctypes as C

from . import FunctionId, Order, Plan, TrigMode
from ._native import check, lib


def shard_rows(total_rows: int, world: int, rank: int):
    """Contiguous, balanced row range of `rank` (first ranks take the
    remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(int(total_rows), int(world))
    count = base + (1 if rank < rem else 0)
    start = rank * base + min(rank, rem)
    return start, count


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (timing)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: torch.Tensor, total_rows: int):
    """Gather every rank's shard (rows) into the full batch on every rank
    (shards are padded to the largest one for the collective)."""
    world = dist.get_world_size()
    counts = [shard_rows(total_rows, world, r)[1] for r in range(world)]
    cmax = max(counts)
    pad = torch.zeros((cmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([parts[r][: counts[r]] for r in range(world)], dim=0)


class ShardedPlan:
    """One Plan per rank over its row shard (weak or strong scaling is the
    caller's choice of total_rows)."""

    def __init__(self, variant: int, n: int, total_rows: int, *, dtype="f32", order=Order.Fast,
                 device: int = 0):
        world = dist.get_world_size() if dist.is_initialized() else 1
        rank = dist.get_rank() if dist.is_initialized() else 0
        self.start, self.rows = shard_rows(total_rows, world, rank)
        self.plan = Plan(variant, FunctionId.Cdft, n, max(1, self.rows), dtype=dtype, order=order,
                         device=device)

    def forward(self, local_in, local_out, stream=None):
        if self.rows:
            self.plan.forward(local_in, local_out, rows=self.rows, stream=stream)


def fourstep_split(n: int):
    """N = n1 * n2 with n1 = 2^ceil(lg N / 2) (the single-GPU four-step's
    split, csrc/fourstep.cu)."""
    lg = int(n).bit_length() - 1
    if n <= 0 or (1 << lg) != n:
        raise ValueError("n must be a power of two")
    n1 = 1 << ((lg + 1) // 2)
    return n1, n // n1


def _plan_covers_f32_fast(n: int) -> bool:
    """Sizes with an fp32 fast-order path: the small-CDFT kernels (2..512),
    the fused kernel (1024..8192) and the single-GPU four-step over them
    (column mode where the first factor is small) up to 2^26."""
    return 2 <= n <= (1 << 26)


def dist_split(n: int, world: int):
    """n = n1 * n2 for the distributed four-step: n2 is a fused-kernel size
    (rows after the exchange; 4096 first, the fastest fused size), n1 any
    size with a fast path (the local rows before it; a column-mode
    single-GPU four-step for 2^13..2^19), both divisible by the world size.
    Config 5, N = 2^30: n1 = 2^18 (64 x 4096, column mode), n2 = 2^12."""
    fourstep_split(n)   # power-of-two check
    for n2 in (4096, 8192, 2048, 1024):
        n1 = n // n2
        if n1 * n2 == n and _plan_covers_f32_fast(n1) and n1 % world == 0 and n2 % world == 0:
            return n1, n2
    raise ValueError(f"no distributed four-step split for n={n}, world={world}")


class CudaLocalOps:
    """One rank's device work for DistFourStep: the fused AM-QFT kernel on
    rows of length n1 and n2, the twiddle+scatter kernel and the transpose
    (C ABI amqft_dist_twiddle_scatter / amqft_transpose_c64)."""

    def __init__(self, variant, n, n1, n2, world, device, trig_mode=TrigMode.Precomputed):
        self.n, self.n1, self.n2 = n, n1, n2
        self.trig_mode = int(trig_mode)
        # the local sub-plans use the same twiddle set (a four-step's own twiddles)
        self.p1 = Plan(variant, FunctionId.Cdft, n1, n2 // world, dtype="f32", order=Order.Fast,
                       device=device, trig_mode=trig_mode, transposable=True)
        self.p2 = Plan(variant, FunctionId.Cdft, n2, n1 // world, dtype="f32", order=Order.Fast,
                       device=device, trig_mode=trig_mode)

        # a column-mode four-step for n1 leaves its rows transposed and the
        # scatter reads them in that order (its final transpose folded in)
        fa = C.c_size_t(0)
        check(lib().amqft_plan_transposed_factor(self.p1._h, C.byref(fa)))
        w = n1 // world
        self.a_t = fa.value if (fa.value and fa.value % 32 == 0 and (n1 // fa.value) % 32 == 0 and w % 32 == 0
                                and n2 // world <= 65535) else 0

    def dft_rows1(self, a, stream=None):
        if self.a_t:
            check(lib().amqft_exec_rows_transposed(self.p1._h, int(a.data_ptr()), int(a.data_ptr()),
                                                   a.shape[0], Plan._stream(stream)))
        else:
            self.p1.forward(a, a, stream=stream)

    def twiddle_scatter(self, a, dst_ptrs, rows, row0, src, nparts, stream=None):
        arr = (C.c_void_p * nparts)(*[int(p) for p in dst_ptrs])
        if self.a_t:
            check(lib().amqft_dist_twiddle_scatter_t(int(a.data_ptr()), arr, rows, self.n1, self.n, row0, src,
                                                     nparts, self.trig_mode, self.a_t, Plan._stream(stream)))
        else:
            check(lib().amqft_dist_twiddle_scatter(int(a.data_ptr()), arr, rows, self.n1, self.n, row0, src,
                                                   nparts, self.trig_mode, Plan._stream(stream)))

    def direct_ok(self, rows):
        """The direct scatter's tiling: 32 x 32 tiles over (rows, kb)."""
        a = self.a_t or 1
        return rows % 32 == 0 and (self.n1 // a) % 32 == 0 and rows // 32 <= 65535

    def twiddle_scatter_direct(self, a, dst_ptrs, rows, row0, nparts, stream=None):
        """Scatter + exchange-side transpose in one kernel: straight into the
        destination ranks' [n1/P][n2] row buffers (amqft_dist_twiddle_scatter_direct)."""
        arr = (C.c_void_p * nparts)(*[int(p) for p in dst_ptrs])
        check(lib().amqft_dist_twiddle_scatter_direct(int(a.data_ptr()), arr, rows, self.n1, self.n, row0, nparts,
                                                      self.trig_mode, self.a_t, Plan._stream(stream)))

    def transpose(self, inp, out, r, c, stream=None):
        check(lib().amqft_transpose_c64(int(inp.data_ptr()), int(out.data_ptr()), 1, r, c,
                                        Plan._stream(stream)))

    def dft_rows2(self, b, z, stream=None):
        self.p2.forward(b, z, stream=stream)


class DistFourStep:
    """Distributed four-step CDFT of one length-N signal over the process
    group (BASELINE config 5).

    n = n1 n2, x viewed as M[n1][n2] = x[n2_total * i1 + i2].  Rank p owns the
    column slab i2 in [p n2/P, (p+1) n2/P) stored as rows of length n1
    (`local_input`).  forward():
      1. length-n1 AM-QFT on the n2/P local rows (fused kernel);
      2. twiddle w_N^(i2 k1) + scatter by k1-slab (one kernel), into the
         send slots -- or, with `peer_recv`, straight into the peers'
         receive buffers over NVLink (the stores are the exchange);
      3. one all-to-all (NCCL) unless step 2 already delivered;
      4. transpose [n2][n1/P] -> [n1/P][n2];
      5. length-n2 AM-QFT on the n1/P rows.
    The output of rank p is X[k1 + n1 k2] for k1 in [p n1/P, (p+1) n1/P),
    as rows k1 of length n2 (`global_output` reassembles it).  One exchange:
    a second all-to-all for natural-order output slabs is not done."""

    def __init__(self, variant: int, n: int, *, group=None, device=None, trig_mode=TrigMode.Precomputed,
                 ops=None, world: int | None = None, rank: int | None = None):
        self.group = group
        self.world = world if world is not None else (dist.get_world_size(group) if dist.is_initialized() else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group) if dist.is_initialized() else 0)
        self.n = int(n)
        self.n1, self.n2 = dist_split(self.n, self.world)
        P = self.world
        if self.n1 % P or self.n2 % P:
            raise ValueError("n1 and n2 must be divisible by the world size")
        self.rows1 = self.n2 // P          # local rows of length n1
        self.w = self.n1 // P              # k1 slab width
        self.device = device
        self.ops = ops if ops is not None else CudaLocalOps(variant, self.n, self.n1, self.n2, P,
                                                            device if device is not None else 0, trig_mode)

    # ---- layout helpers (host side)
    def local_input(self, x_full):
        """Rank's slab from a full interleaved (re, im) signal: [n2/P][2 n1]."""
        P, p = self.world, self.rank
        xc = x_full.reshape(self.n1, self.n2, 2)
        cols = xc[:, p * self.rows1:(p + 1) * self.rows1, :]
        if hasattr(cols, "permute"):
            return cols.permute(1, 0, 2).reshape(self.rows1, 2 * self.n1).contiguous()
        return cols.transpose(1, 0, 2).reshape(self.rows1, 2 * self.n1).copy()

    def global_output(self, parts):
        """Natural-order X (interleaved) from every rank's [n1/P][2 n2] output."""
        import numpy as np
        X = np.empty((self.n2, self.n1, 2), dtype=np.asarray(parts[0]).dtype)
        for q, z in enumerate(parts):
            zc = np.asarray(z).reshape(self.w, self.n2, 2)
            X[:, q * self.w:(q + 1) * self.w, :] = zc.transpose(1, 0, 2)
        return X.reshape(-1)

    def buffers(self, like):
        """send, recv, b, z buffers for forward()."""
        P = self.world
        send = like.new_empty((P, self.rows1 * self.w * 2))
        recv = like.new_empty((P, self.rows1 * self.w * 2))
        b = like.new_empty((self.w, 2 * self.n2))
        z = like.new_empty((self.w, 2 * self.n2))
        return send, recv, b, z

    def map_peer_rows(self, b):
        """Every rank's `b` row buffer (bufs[2]) mapped into this process: the
        `peer_rows` list of forward()'s direct mode.  The buffers travel as
        CUDA IPC handles (torch's shared-storage reduction, cudaIpcGetMemHandle
        / cudaIpcOpenMemHandle underneath) over the process group, so the ranks
        may be separate processes -- on NVLink-connected GPUs of one node, or
        on one GPU.  Collective; the mapped tensors are kept alive on self."""
        from torch.multiprocessing.reductions import reduce_tensor
        if self.world == 1 or not dist.is_initialized():
            self._peer_row_tensors = [b]
            return [b.data_ptr()]
        handles = [None] * self.world
        dist.all_gather_object(handles, reduce_tensor(b), group=self.group)
        self._peer_row_tensors = [b if q == self.rank else fn(*args) for q, (fn, args) in enumerate(handles)]
        return [t.data_ptr() for t in self._peer_row_tensors]

    def stage1(self, a, send, peer_recv=None, stream=None):
        """Length-n1 transforms of the local rows, then twiddle + scatter by
        k1-slab into the send slots, or into the peers' receive buffers."""
        P, p = self.world, self.rank
        self.ops.dft_rows1(a, stream)
        row0 = p * self.rows1
        if peer_recv is not None:
            self.ops.twiddle_scatter(a, peer_recv, self.rows1, row0, p, P, stream)
        else:
            base = int(send.data_ptr())
            slot = self.rows1 * self.w * 2 * a.element_size()
            self.ops.twiddle_scatter(a, [base + q * slot for q in range(P)], self.rows1, row0, 0, P, stream)

    def stage2(self, recv, b, z, stream=None):
        """recv = [n2][n1/P] (complex) -> transpose -> length-n2 transforms."""
        self.ops.transpose(recv, b, self.n2, self.w, stream)
        self.ops.dft_rows2(b, z, stream)
        return z

    def forward(self, a, bufs=None, peer_recv=None, stream=None, peer_rows=None):
        """a: this rank's [n2/P][2 n1] slab (overwritten).  Returns z, this
        rank's [n1/P][2 n2] output slab.

        peer_rows: every rank's `b` row buffer ([n1/P][2 n2], bufs[2]) mapped
        into this process: the scatter writes each value straight to its
        final place there (scatter + exchange + transpose in one kernel, the
        "direct" mode).  With one rank the mode is the default: the rank's own
        buffer, no exchange to make."""
        send, recv, b, z = bufs if bufs is not None else self.buffers(a)
        multi = self.world > 1 and dist.is_initialized()
        direct = getattr(self.ops, "direct_ok", None)
        if peer_rows is None and self.world == 1 and peer_recv is None and direct and direct(self.rows1):
            peer_rows = [b.data_ptr()]
        if peer_rows is not None:
            if multi:   # write-after-read on the peers' row buffers
                if a.is_cuda:
                    torch.cuda.synchronize(a.device)
                dist.barrier(group=self.group)
            self.ops.dft_rows1(a, stream)
            self.ops.twiddle_scatter_direct(a, peer_rows, self.rows1, self.rank * self.rows1, self.world, stream)
            if multi:   # the stores were the exchange: order them before the peers read
                if a.is_cuda:
                    torch.cuda.synchronize(a.device)
                dist.barrier(group=self.group)
            self.ops.dft_rows2(b, z, stream)
            return z
        if peer_recv is not None and multi:
            # write-after-read: no rank may scatter into a peer's receive
            # buffer while that peer still transposes the previous call's data
            if a.is_cuda:
                torch.cuda.synchronize(a.device)
            dist.barrier(group=self.group)
        self.stage1(a, send, peer_recv, stream)
        if peer_recv is not None:
            # the scatter's stores were the exchange; order them before the
            # peers read their receive buffers
            if multi:
                if a.is_cuda:
                    torch.cuda.synchronize(a.device)
                dist.barrier(group=self.group)
        elif self.world > 1:
            # the collective runs on the caller's stream, after the scatter
            if a.is_cuda and stream is not None:
                with torch.cuda.stream(stream):
                    dist.all_to_all_single(recv, send, group=self.group)
            else:
                dist.all_to_all_single(recv, send, group=self.group)
        else:
            recv = send   # one part: the scatter already produced the layout
        return self.stage2(recv, b, z, stream)


class DistPlan:
    """The distributed four-step behind the C ABI (amqft_dist_*, csrc/dist.cpp):
    one plan per rank owning its NCCL communicator, the same slab layouts as
    DistFourStep.  Rank 0 makes the NCCL unique id; it reaches the other ranks
    over the torch.distributed group (any backend).  With one rank and
    use_nccl=False there is no communicator."""

    def __init__(self, variant: int, n: int, *, device: int = 0, trig_mode=TrigMode.Precomputed, group=None,
                 world: int | None = None, rank: int | None = None, use_nccl: bool = True):
        self.world = world if world is not None else (dist.get_world_size(group) if dist.is_initialized() else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group) if dist.is_initialized() else 0)
        uid = None
        if use_nccl or self.world > 1:
            buf = (C.c_ubyte * 128)()
            if self.rank == 0:
                check(lib().amqft_dist_unique_id(buf))
            if self.world > 1:
                t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
                obj = [t]
                dist.broadcast_object_list(obj, src=0, group=group)
                buf = (C.c_ubyte * 128)(*obj[0].tolist())
            uid = buf
        self._h = C.c_void_p()
        check(lib().amqft_dist_plan_create(C.byref(self._h), int(variant), int(n), int(self.world), int(self.rank),
                                           int(device), int(trig_mode), uid))
        a, b, c, d = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_size_t()
        check(lib().amqft_dist_plan_shape(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        self.n, self.n1, self.n2, self.rows_in, self.rows_out = int(n), a.value, b.value, c.value, d.value

    def forward(self, slab, out, stream=None):
        """slab: [n2/P][2 n1] fp32 (overwritten); out: [n1/P][2 n2]."""
        check(lib().amqft_dist_exec_forward(self._h, int(slab.data_ptr()), int(out.data_ptr()), Plan._stream(stream)))
        return out

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().amqft_dist_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
