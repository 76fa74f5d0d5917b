"""Probe: can two processes form an NCCL communicator on the same GPU (this NCCL build)?"""
import os
import sys

import torch
import torch.distributed as dist


def main():
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    x = torch.ones(4, device="cuda") * (rank + 1)
    try:
        dist.all_reduce(x)
        torch.cuda.synchronize()
        print("rank", rank, "allreduce ok", x.tolist(), flush=True)
    except Exception as e:  # noqa: BLE001
        print("rank", rank, "failed:", repr(e)[:300], flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
