"""dev: all-gather of per-rank slabs by copy-engine pulls from CUDA-IPC-mapped
peer buffers (torchrun, one process per GPU), vs NCCL all_gather_into_tensor.
  torchrun --nproc-per-node N tools/ipc_bw.py [MB per rank]"""
import os, sys, time
import torch, torch.distributed as dist
from cuda.bindings import runtime as rt

def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    assert int(err) == 0, r
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None

dist.init_process_group("nccl")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(rank)
mb = float(sys.argv[1]) if len(sys.argv) > 1 else 18.4
nbytes = int(mb * 1e6) // 512 * 512
win = ck(rt.cudaMalloc(nbytes))
dst = ck(rt.cudaMalloc(nbytes * world))
ck(rt.cudaMemset(win, rank + 1, nbytes))
h = ck(rt.cudaIpcGetMemHandle(win))
hb = bytes(h.reserved)
allh = [None] * world
dist.all_gather_object(allh, hb)
peers = {}
for p in range(world):
    if p == rank:
        continue
    hh = rt.cudaIpcMemHandle_t()
    hh.reserved = allh[p]
    peers[p] = ck(rt.cudaIpcOpenMemHandle(hh, rt.cudaIpcMemLazyEnablePeerAccess))
streams = [ck(rt.cudaStreamCreateWithFlags(rt.cudaStreamNonBlocking)) for _ in range(world)]
def pull():
    for p, ptr in peers.items():
        ck(rt.cudaMemcpyAsync(int(dst) + p * nbytes, ptr, nbytes, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice, streams[p]))
    for p in peers:
        ck(rt.cudaStreamSynchronize(streams[p]))
for _ in range(3):
    pull()
dist.barrier(); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    pull()
dt = (time.perf_counter() - t) / 20
x = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
y = torch.empty(world * nbytes // 8, dtype=torch.float64, device="cuda")
for _ in range(3):
    dist.all_gather_into_tensor(y, x)
torch.cuda.synchronize(); dist.barrier()
t = time.perf_counter()
for _ in range(20):
    dist.all_gather_into_tensor(y, x)
torch.cuda.synchronize()
dn = (time.perf_counter() - t) / 20
if rank == 0:
    print(f"{world} GPUs, {nbytes/1e6:.1f} MB per rank: IPC CE pulls {dt*1e6:.1f} us "
          f"({(world-1)*nbytes/dt/1e9:.0f} GB/s in), NCCL allgather {dn*1e6:.1f} us "
          f"({(world-1)*nbytes/dn/1e9:.0f} GB/s in)", flush=True)
dist.barrier()
for ptr in peers.values():
    ck(rt.cudaIpcCloseMemHandle(ptr))
dist.destroy_process_group()
