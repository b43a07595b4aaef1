"""NCCL allreduce bus bandwidth on this box (SURVEY.md §8e asks for it before relying on the
gradient-allreduce cost estimate).  torchrun --nproc-per-node N scripts/allreduce_sweep.py
Prints one JSON line per size (rank 0): bytes, ms (CUDA events, median of 10), algorithm
bandwidth and bus bandwidth = algbw * 2 (N-1) / N."""
import json
import os

import torch
import torch.distributed as dist


def main():
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    n = dist.get_world_size()
    for mb in (1, 16, 64, 256, 1024, 2048):
        x = torch.ones(mb * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
        for _ in range(3):
            dist.all_reduce(x)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            a.record()
            dist.all_reduce(x)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = torch.tensor([sorted(ts)[len(ts) // 2]], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        byts = x.numel() * 4
        algbw = byts / (ms / 1e3) / 1e9
        if dist.get_rank() == 0:
            print(json.dumps({"n_gpus": n, "bytes": byts, "ms": ms, "algbw_gbs": algbw,
                              "busbw_gbs": algbw * 2 * (n - 1) / n}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
