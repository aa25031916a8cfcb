"""World-size-2 gloo tests of the multi-GPU host logic (no GPU needed).

The data path shards rows with no collective; these tests check the shard
partition, the max-over-ranks timing reduction and the row gather, with the
CPU oracle standing in for each rank's device transform (test-only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1404_1810_b200.dist import gather_rows, max_over_ranks, shard_rows


def test_shard_rows_partition():
    for total in (0, 1, 7, 65536, 65537):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                s, c = shard_rows(total, world, r)
                seen.extend(range(s, s + c))
            assert seen == list(range(total))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import oracle as O
    r = O.restatement()
    rng = np.random.default_rng(3)
    full = rng.standard_normal((total, 2 * n))
    start, cnt = shard_rows(total, world, rank)
    local = np.stack([r.execute(4, O.F_CDFT, n, full[i]) for i in range(start, start + cnt)])
    gathered = gather_rows(torch.tensor(local), total).numpy()
    ms = max_over_ranks(1.0 + rank)
    if rank == 0:
        want = np.stack([r.execute(4, O.F_CDFT, n, full[i]) for i in range(total)])
        q.put((bool(np.array_equal(gathered, want)), ms))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_shard_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 64, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, ms = q.get(timeout=100)
    for p in procs:
        p.join(timeout=60)
    assert ok
    assert ms == 2.0


# ---- distributed four-step (config 5) host logic -----------------------
class NumpyLocalOps:
    """TEST STAND-IN for one rank's device kernels (CudaLocalOps): the same
    index semantics (rows of interleaved fp32 complex, twiddle + scatter by
    k1-slab into raw slot pointers, transpose) with numpy's FFT for the
    local transforms.  Lets the gloo test check the distributed orchestration
    (layouts, all-to-all, output mapping) without a GPU."""

    def __init__(self, n, n1, n2):
        self.n, self.n1, self.n2 = n, n1, n2

    @staticmethod
    def _c(t, rows, cols):
        a = t.numpy().reshape(rows, cols, 2)
        return a[..., 0] + 1j * a[..., 1]

    @staticmethod
    def _put(t, z):
        a = t.numpy().reshape(z.shape + (2,))
        a[..., 0], a[..., 1] = z.real, z.imag

    def dft_rows1(self, a, stream=None):
        rows = a.numel() // (2 * self.n1)
        self._put(a, np.fft.fft(self._c(a, rows, self.n1), axis=1))

    def twiddle_scatter(self, a, dst_ptrs, rows, row0, src, nparts, stream=None):
        import ctypes as C
        w = self.n1 // nparts
        z = self._c(a, rows, self.n1)
        i2 = (row0 + np.arange(rows))[:, None]
        k1 = np.arange(self.n1)[None, :]
        z = z * np.exp(-2j * np.pi * ((i2 * k1) % self.n) / self.n)
        for q in range(nparts):
            blk = z[:, q * w:(q + 1) * w]
            buf = np.ctypeslib.as_array((C.c_float * (2 * rows * w * (src + 1))).from_address(int(dst_ptrs[q])))
            out = buf[2 * src * rows * w:].reshape(rows, w, 2)
            out[..., 0], out[..., 1] = blk.real, blk.imag

    def transpose(self, inp, out, r, c, stream=None):
        self._put(out, self._c(inp, r, c).T.copy())

    def dft_rows2(self, b, z, stream=None):
        rows = b.numel() // (2 * self.n2)
        self._put(z, np.fft.fft(self._c(b, rows, self.n2), axis=1))


def _dist_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1404_1810_b200.dist import DistFourStep, dist_split
    n1, n2 = dist_split(n, world)
    d = DistFourStep(4, n, ops=NumpyLocalOps(n, n1, n2))
    rng = np.random.default_rng(30)
    x = rng.standard_normal(2 * n).astype(np.float32)
    a = d.local_input(torch.tensor(x))
    z = d.forward(a)
    parts = [torch.empty_like(z) for _ in range(world)]
    dist.all_gather(parts, z)
    if rank == 0:
        X = d.global_output([p.numpy() for p in parts]).astype(np.float64)
        f = np.fft.fft(x[0::2].astype(np.float64) + 1j * x[1::2].astype(np.float64))
        ref = np.empty(2 * n)
        ref[0::2], ref[1::2] = f.real, f.imag
        q.put(float(np.linalg.norm(X - ref) / np.linalg.norm(ref)))
    dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_gloo_world2_distributed_fourstep():
    """Config 5 orchestration at world size 2 over gloo: column slabs in,
    one all-to-all, k1-slabs out; reassembled output equals the DFT."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n = 1 << 20
    ps = [ctx.Process(target=_dist_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in ps:
        p.start()
    err = q.get(timeout=170)
    for p in ps:
        p.join(timeout=60)
    assert err < 1e-5, err


def test_dist_split_and_layout_helpers():
    from paper_1404_1810_b200.dist import DistFourStep, dist_split
    assert dist_split(1 << 30, 8) == (1 << 18, 1 << 12)
    assert dist_split(1 << 24, 2) == (4096, 4096)
    with pytest.raises(ValueError):
        dist_split(3 << 20, 2)
    n = 1 << 20
    for world in (1, 2, 4):
        parts = []
        for rank in range(world):
            d = DistFourStep(4, n, ops=object(), world=world, rank=rank)
            x = np.arange(2 * n, dtype=np.float32)
            loc = d.local_input(x)
            assert loc.shape == (d.rows1, 2 * d.n1)
            # local row r, element i1 is x[n2 * i1 + rank * rows1 + r]
            r, i1 = 3, 5
            m = d.n2 * i1 + rank * d.rows1 + r
            assert loc[r, 2 * i1] == x[2 * m]
            parts.append(np.arange(d.w * 2 * d.n2, dtype=np.float64) + rank * 1e7)
        X = DistFourStep(4, n, ops=object(), world=world, rank=0).global_output(parts)
        d = DistFourStep(4, n, ops=object(), world=world, rank=0)
        # X[k1 + n1 k2] comes from rank k1 // w, row k1 % w, column k2
        k1, k2 = d.n1 - 1, 7
        src = parts[k1 // d.w].reshape(d.w, d.n2, 2)[k1 % d.w, k2]
        assert X[2 * (k1 + d.n1 * k2)] == src[0]


def test_dist_plan_c_abi_rejects_bad_requests():
    """amqft_dist_plan_create validates before touching a device or NCCL."""
    import ctypes as C
    from paper_1404_1810_b200 import _native
    L = _native.lib()
    h = C.c_void_p()
    for args in ((4, 1 << 20, 0, 0), (4, 1 << 20, 2, 2), (4, 3 << 20, 1, 0), (4, 1 << 20, 2, 0)):
        v, n, parts, rank = args
        s = L.amqft_dist_plan_create(C.byref(h), v, n, parts, rank, 0, 0, None)
        assert s == _native.EINVAL, args
