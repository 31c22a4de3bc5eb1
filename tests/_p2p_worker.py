"""Worker for the GPU test of the p2p combine: several processes on ONE GPU exchange CUDA IPC
mappings (the same mechanism as peer GPUs over NVLink; host-side gloo barriers order the
levels, so no kernel waits on another process's kernel)."""
import os


def run(rank, world, port, cfg, q):
    import numpy as np
    import torch
    import torch.distributed as dist

    import ddqd_inputs as gen
    from paper_1510_08642_b200.mgpu import DistributedGemm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, algo, T, m, l, n, k = cfg
        dev = torch.device("cuda", 0)
        A = torch.from_numpy(gen.matrix(W, m, l, 31, 0)).to(dev)
        B = torch.from_numpy(gen.matrix(W, l, n, 31, 1)).to(dev)
        C = torch.zeros((W, m, n), dtype=torch.float64, device=dev)
        dg = DistributedGemm(W, algo, T, m, l, n, dist, dev, k=k, combine="p2p", replicated_inputs=True)
        dg(A, B, C)
        dg(A, B, C)   # mappings and buffers reused
        torch.cuda.synchronize()
        if rank == 0:
            q.put((dg.k, C.cpu().numpy().copy()))
        dg.release()
    except Exception as e:   # surface the failure to the parent
        q.put(("error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()
