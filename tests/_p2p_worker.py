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


def run_schedules(rank, world, port, cfg, q):
    """Every multi-GPU schedule's CUDA path with `world` processes on ONE GPU, exchanges over
    gloo staged through host memory (mgpu.HostStagedGroup; no kernel waits on another process):
    the band schedule, the depth-k products with the NCCL-style combine on rank 0 and with the
    p2p combine, the automatic choice, and the band schedule with beta = 1."""
    import torch
    import torch.distributed as tdist

    import ddqd_inputs as gen
    from paper_1510_08642_b200 import mgpu

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    dist = mgpu.HostStagedGroup(tdist)
    try:
        W, algo, T, m, l, n = cfg
        dev = torch.device("cuda", 0)

        def inputs():
            if rank == 0:
                return (torch.from_numpy(gen.matrix(W, m, l, 33, 0)).to(dev),
                        torch.from_numpy(gen.matrix(W, l, n, 33, 1)).to(dev))
            return (torch.zeros((W, m, l), dtype=torch.float64, device=dev),
                    torch.zeros((W, l, n), dtype=torch.float64, device=dev))

        out = {}
        for name, mk in (("bands", lambda: mgpu.BandGemm(W, algo, T, m, l, n, dist, dev)),
                         ("products", lambda: mgpu.DistributedGemm(W, algo, T, m, l, n, dist, dev)),
                         ("products_p2p", lambda: mgpu.DistributedGemm(W, algo, T, m, l, n, dist, dev,
                                                                       combine="p2p")),
                         ("products_rows", lambda: mgpu.DistributedGemm(W, algo, T, m, l, n, dist, dev,
                                                                        combine="rows")),
                         ("auto", lambda: mgpu.AutoDistributedGemm(W, algo, T, m, l, n, dist, dev))):
            A, B = inputs()
            C = torch.zeros((W, m, n), dtype=torch.float64, device=dev)
            s = mk()
            s(A, B, C)
            s(A, B, C)
            torch.cuda.synchronize()
            if hasattr(s, "release"):
                s.release()
            out[name] = C.cpu().numpy().copy()
        A, B = inputs()
        C = torch.from_numpy(gen.matrix(W, m, n, 33, 2)).to(dev) if rank == 0 else None
        mgpu.BandGemm(W, algo, T, m, l, n, dist, dev, beta=1)(A, B, C)
        torch.cuda.synchronize()
        if rank == 0:
            out["bands_beta1"] = C.cpu().numpy().copy()
        A, B = inputs()
        C = torch.from_numpy(gen.matrix(W, m, n, 33, 2)).to(dev) if rank == 0 else None
        mgpu.DistributedGemm(W, algo, T, m, l, n, dist, dev, beta=1, combine="rows")(A, B, C)
        torch.cuda.synchronize()
        if rank == 0:
            out["rows_beta1"] = C.cpu().numpy().copy()
            q.put(out)
    except Exception as e:   # surface the failure to the parent
        q.put({"error": repr(e)})
        raise
    finally:
        tdist.destroy_process_group()
