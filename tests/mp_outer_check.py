"""Multi-GPU parity worker (launched by tests/test_multigpu_gpu.py under
torchrun): one Pier group per GPU, the checks of tests/group_checks.py
(`outer_checks`) on a real NCCL / NVLink communicator; rank 0 writes the JSON.
The same checks run on one GPU as a VirtualGroup (tests/test_virtual_groups_gpu.py)."""

import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2511_17849_b200 as P  # noqa: E402
from group_checks import outer_checks  # noqa: E402


def main():
    out_path = sys.argv[1]
    bucket = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = P.GroupComm(rank, world)
    res = outer_checks(comm, bucket)
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump(res, fh)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
