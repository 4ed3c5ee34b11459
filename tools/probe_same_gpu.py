"""Probe: what multi-process collectives work with 2 ranks on ONE GPU (the gpurun box has one)?
  1. torch NCCL process group world=2 on the same device (NCCL normally rejects duplicate GPUs)
  2. CUDA IPC of a device buffer between two processes on the same device (cudaIpcOpenMemHandle)
  3. cross-process device-side flag spin (time-sliced contexts): does a spinning kernel make progress?"""
import os
import sys
import time

import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def nccl_probe(rank, world, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = "29533"
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("nccl", rank=rank, world_size=world)
        t = torch.ones(4, device="cuda") * (rank + 1)
        dist.all_reduce(t)
        torch.cuda.synchronize()
        q.put((rank, "nccl ok", t.tolist()))
    except Exception as e:
        q.put((rank, "nccl fail", repr(e)[:400]))
    finally:
        try:
            dist.destroy_process_group()
        except Exception:
            pass


def ipc_probe(rank, world, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = "29534"
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        buf = torch.full((1024,), float(rank + 10), device="cuda")
        # share via torch's IPC (cudaIpcGetMemHandle under the hood)
        from torch.multiprocessing.reductions import reduce_tensor
        h = reduce_tensor(buf)
        objs = [None] * world
        dist.all_gather_object(objs, (h[0], h[1]))
        peer = (rank + 1) % world
        if objs[peer] is None:
            raise RuntimeError("no handle")
        fn, args = objs[peer]
        t = fn(*args)
        q.put((rank, "ipc ok", float(t[0].item())))
        dist.barrier()
    except Exception as e:
        q.put((rank, "ipc fail", repr(e)[:400]))
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.set_start_method("spawn")
    for fn in (nccl_probe, ipc_probe):
        q = mp.Queue()
        ps = [mp.Process(target=fn, args=(r, 2, q)) for r in range(2)]
        for p in ps:
            p.start()
        t0 = time.time()
        for p in ps:
            p.join(timeout=90)
        for p in ps:
            if p.is_alive():
                p.kill()
                print(fn.__name__, "timeout")
        while not q.empty():
            print(fn.__name__, q.get())
        print(fn.__name__, "took", round(time.time() - t0, 1), "s", flush=True)
