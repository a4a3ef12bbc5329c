"""Multi-GPU worker for groups x dp x tp layouts,
launched by tests/test_multigpu_gpu.py under torchrun with 4 ranks: the
`topology_checks` of tests/group_checks.py (layouts 2x2x1 and 2x1x2) on a real
communicator; rank 0 writes the JSON.  The same checks, plus 2x2x2 on eight
ranks, run on one GPU as VirtualGroups (tests/test_virtual_groups_gpu.py)."""

import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2511_17849_b200 as P  # noqa: E402
from group_checks import topology_checks  # noqa: E402


def main():
    out_path = sys.argv[1]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    comm = P.GroupComm(rank, world)
    res = topology_checks(comm, ("dp2", "tp2"))
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump(res, fh)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
