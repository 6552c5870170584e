"""Multi-GPU layer (one process per GPU, torch.distributed for the plumbing).

Partition:
- full->band is distributed inside the library over a collective context
  (skew_ctx_create_dist): 1D block-cyclic 64-wide column blocks (owner of block q = q mod P),
  the owner factors each panel and NCCL-broadcasts V / T / tau, every rank forms its partial
  skew-SYMM product from its own column blocks, the partials are summed with an allreduce,
  W is formed redundantly and each rank applies the rank-2k update to its own column blocks;
- the band is combined with one allreduce and the bulge chase runs replicated (deterministic,
  bit-identical on every rank);
- the multisection eigenvalue search is sharded by task slice plus an allgather;
- the eigenpairs are split into contiguous index ranges [k0, k1) per rank: inverse
  iteration (with ghost vectors for the re-orthogonalisation window), D assembly, BT2 and BT1
  on the rank's 2*(k1-k0) columns of [Re | Im], with no data-path collective (PAPER.md:336-338:
  "applied on the real and imaginary part independently").
Gathering the vectors (optional, for callers that want them on one rank) is a plain
all_gather.  The same distributed code runs on one GPU through virtual ranks
(Context(virtual=...), tests/test_gpu_virtual_ranks.py).
"""
import os

__all__ = ["eigpair_range", "init_from_env", "skew_eig_distributed", "gather_columns"]


def eigpair_range(nev, rank, world):
    """Contiguous, balanced eigenpair index range [k0, k1) of `rank` out of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return (rank * nev) // world, ((rank + 1) * nev) // world


def init_from_env(backend="nccl"):
    """Initialise torch.distributed from RANK / WORLD_SIZE / LOCAL_RANK / MASTER_* (torchrun)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def skew_eig_distributed(A, nev=None, group=None, ctx=None, overwrite_a=False):
    """Per-rank solve: returns (lam (all nev), Zre_local, Zim_local, k0, k1) with the local
    eigenvectors z_{k0} .. z_{k1-1} of the rank's range."""
    import torch.distributed as dist
    from . import skew_eig_range
    n = A.shape[0]
    nev = n // 2 if nev is None else nev
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    k0, k1 = eigpair_range(nev, rank, world)
    lam, Zre, Zim = skew_eig_range(A, nev, k0, k1, ctx=ctx, overwrite_a=overwrite_a)
    return lam, Zre, Zim, k0, k1


def gather_columns(local, nev, group=None):
    """all_gather the column blocks (n x (k1-k0) per rank, ranges from eigpair_range) into the
    full n x nev matrix on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = local.shape[0]
    width = max(k1 - k0 for k0, k1 in (eigpair_range(nev, r, world) for r in range(world)))
    buf = torch.zeros((width, n), dtype=local.dtype, device=local.device)
    buf[: local.shape[1]] = local.t()
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    cols = []
    for r in range(world):
        k0, k1 = eigpair_range(nev, r, world)
        cols.append(parts[r][: k1 - k0])
    return torch.cat(cols, dim=0).t()
