"""Multi-process helpers of the tier-split tests: file-based rendezvous (no TCP port to race for)
and rank processes that are always reaped, so a failing or hung rank can never keep the test
session alive."""
import os
import tempfile


def rendezvous() -> str:
    """A fresh path for torch.distributed's file store (init_method file://)."""
    fd, path = tempfile.mkstemp(prefix="gh_rdv_")
    os.close(fd)
    os.unlink(path)
    return path


def init_rank(rank: int, world: int, rdv: str) -> None:
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method="file://" + rdv, rank=rank, world_size=world)


def spawn(target, world: int, args=()):
    """Start `world` daemon processes target(rank, world, rdv, q, *args); returns (procs, q)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    rdv = rendezvous()
    procs = [ctx.Process(target=target, args=(r, world, rdv, q) + tuple(args), daemon=True) for r in range(world)]
    for p in procs:
        p.start()
    return procs, q


def collect(procs, q, n: int = 1, timeout: float = 600):
    """n results from the queue, then every rank's clean exit; kills the ranks on any failure."""
    try:
        out = [q.get(timeout=timeout) for _ in range(n)]
        for p in procs:
            p.join(timeout=120)
            assert p.exitcode == 0, f"rank process exited with {p.exitcode}"
        return out
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
                p.join(timeout=10)
