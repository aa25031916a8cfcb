"""Worker of tests/test_gpu_dist_ipc.py: one rank of a world-2 distributed
four-step whose ranks are SEPARATE PROCESSES sharing one GPU.  The direct
mode's peer row buffers are mapped with CUDA IPC (DistFourStep.map_peer_rows);
the only synchronisation is host-side (gloo barriers around the scatter), no
kernel waits on another process.  Launched by torch.distributed.run."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1404_1810_b200.dist import DistFourStep  # noqa: E402


def main():
    out_path = sys.argv[1]
    n = 1 << int(sys.argv[2])
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    x = np.random.default_rng(77).standard_normal(2 * n).astype(np.float32)   # the same signal on every rank
    d = DistFourStep(4, n, device=0)
    a = d.local_input(torch.tensor(x)).to("cuda:0")
    bufs = d.buffers(a)
    rows = d.map_peer_rows(bufs[2])
    assert len(rows) == world and rows[rank] == bufs[2].data_ptr()
    z = d.forward(a, bufs=bufs, peer_rows=rows)
    torch.cuda.synchronize()
    # a second call on the same buffers (write-after-read across the processes)
    a2 = d.local_input(torch.tensor(x)).to("cuda:0")
    z = d.forward(a2, bufs=bufs, peer_rows=rows)
    torch.cuda.synchronize()
    parts = [None] * world
    dist.all_gather_object(parts, z.cpu().numpy())
    if rank == 0:
        got = d.global_output(parts).astype(np.float64)
        f = np.fft.fft(x[0::2].astype(np.float64) + 1j * x[1::2].astype(np.float64))
        ref = np.empty(2 * n)
        ref[0::2], ref[1::2] = f.real, f.imag
        err = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        np.save(out_path, np.array([err]))
    # unmap the peers' buffers before any process frees its own (torch's CUDA IPC reference
    # counting), then leave without the interpreter's teardown of the IPC machinery
    d._peer_row_tensors = None
    del rows, z, bufs, a, a2
    import gc
    gc.collect()
    torch.cuda.ipc_collect()
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()
    sys.stdout.flush()
    os._exit(0)


if __name__ == "__main__":
    main()
