"""Probe of the CUDA IPC plumbing behind peer.py (bc_ipc_export / bc_ipc_open and
interprocess events) with two processes on cuda:0: values written by one process
are read by the other through the mapping, both directions, with a kernel in
between ordered by an IPC event.  Prints one line per check."""
import os
import socket
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def work(rank, port):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from paper_2309_04909_b200 import api
    pad = torch.zeros(1000, dtype=torch.int64, device="cuda")  # so the buffer is not at its segment's start
    buf = torch.arange(4096, dtype=torch.int64, device="cuda") * (rank + 1)
    ev = torch.cuda.Event(interprocess=True)
    h, off = api.ipc_export(buf)
    blobs = [None, None]
    dist.all_gather_object(blobs, (h, off, bytes(ev.ipc_handle())))
    ph, poff, pev = blobs[1 - rank]
    base = api.ipc_open(ph)
    peer = api.tensor_at(base + poff, (4096,), torch.int64)
    print(f"rank {rank}: own ptr {buf.data_ptr():#x} off {off}, peer mapped at {base:#x}+{poff} device {peer.device}",
          flush=True)
    got = peer.clone()
    torch.cuda.synchronize()
    exp = torch.arange(4096, dtype=torch.int64, device="cuda") * (2 - rank)
    print(f"rank {rank}: read peer {'OK' if torch.equal(got, exp) else 'MISMATCH ' + str(got[:4].tolist())}", flush=True)
    dist.barrier()
    # rank 0 writes into rank 1's buffer with a kernel, records the event, rings; rank 1 waits on the event
    if rank == 0:
        torch.cuda._sleep(200_000_000)  # make the write late: only the event orders it
        peer.fill_(7)
        ev.record()
        dist.send(torch.zeros(1), 1)
    else:
        dist.recv(torch.zeros(1), 0)
        pe = torch.cuda.Event.from_ipc_handle(torch.device("cuda", 0), pev)
        torch.cuda.current_stream().wait_event(pe)
        v = buf.clone()
        torch.cuda.synchronize()
        print(f"rank 1: event-ordered read {'OK' if bool((v == 7).all()) else 'STALE ' + str(v[:4].tolist())}",
              flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    api.ipc_close(base)
    dist.barrier()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(work, args=(port,), nprocs=2, join=True, start_method="spawn")
