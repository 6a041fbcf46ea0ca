"""Worker of tests/test_gpu_parity.py::test_nccl_two_ranks_equals_local_ranks (run under
torch.distributed.run, one process per GPU): the NCCL row-block solve of cfg3 (halo-AINV w and
the plain one; optional pcg flags, e.g. PCG_FLAG_DEVICE_COMM), written by rank 0 as .npz for the test to compare with the one-GPU local-ranks
emulation and the oracle's partitioned canonical PCG."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1210_1878_b200 as pcg  # noqa: E402
from paper_1210_1878_b200 import synth  # noqa: E402


def main():
    out, name, w = sys.argv[1], sys.argv[2], int(sys.argv[3])
    flags = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    p = synth.config(name)
    b = np.load(out + ".b.npy")
    S = pcg.Solver(p.cE, p.cN, p.mask, tau=0.1 + 1e-9, ainv_halo=w, group=dist.group.WORLD, device=local, flags=flags)
    bd = torch.from_numpy(np.ascontiguousarray(b[S.j_begin:S.j_end])).cuda()
    x, k, hist, rep = S.solve(bd, tol=1e-10)
    parts = [None] * world
    dist.all_gather_object(parts, x.cpu().numpy())
    if rank == 0:
        np.savez(out, x=np.concatenate(parts, axis=0), k=k, hist=hist, driver=rep["driver"],
                 true_rel=rep["true_rel_residual"])
    S.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
