"""Exchange ceiling on this node (context for the NVLink roofline).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port 29531 profiles/nvlink_sweep.py

NCCL all_to_all_single over NVLink/NVSwitch for 1 MB .. 1 GB per rank, and a plain
peer-to-peer copy (cudaMemcpyPeer via torch .copy_ between devices of one process is
not available with one process per GPU, so the P2P figure is the NCCL send/recv pair).
Device time, max over ranks.  Prints one JSON line on rank 0.
"""
import json
import os

import torch
import torch.distributed as dist


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    out = []
    for mb in (1, 16, 64, 256, 1024):
        n = mb * (1 << 20) // 4
        n -= n % world
        x = torch.ones(n, dtype=torch.float32, device="cuda")
        y = torch.empty_like(x)
        ms = timed(lambda: dist.all_to_all_single(y, x))
        sent = 4 * n * (world - 1) / world          # bytes leaving each GPU
        out.append({"MB_per_rank": mb, "ms": ms, "GBps_out_per_gpu": sent / (ms / 1e3) / 1e9})
    if world >= 2:
        n = 256 * (1 << 20) // 4
        x = torch.ones(n, dtype=torch.float32, device="cuda")

        def pair():
            if rank == 0:
                dist.send(x, 1)
            elif rank == 1:
                dist.recv(x, 0)
        ms = timed(pair)
        p2p = {"MB": 256, "ms": ms, "GBps": 4 * n / (ms / 1e3) / 1e9}
    else:
        p2p = None
    if rank == 0:
        print(json.dumps({"world": world, "nccl_all_to_all": out, "nccl_send_recv_0_to_1": p2p,
                          "nominal_GBps_per_direction": 900}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
