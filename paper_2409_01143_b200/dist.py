"""Process-group plumbing: one process per GPU, NCCL id exchange through the
torch.distributed TCPStore (torch is plumbing only; the step runs in
libhexexec.so).  Reads RANK / WORLD_SIZE / LOCAL_RANK / MASTER_ADDR /
MASTER_PORT like torchrun sets them."""
from __future__ import annotations

import datetime
import os

from .hexexec import Executor, unique_id


def env_rank():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


_STORE = None


def store(rank: int, world: int):
    """TCPStore shared by all ranks (rank 0 hosts it)."""
    global _STORE
    if _STORE is None and world > 1:
        import torch.distributed as td
        addr = os.environ.get("MASTER_ADDR", "127.0.0.1")
        port = int(os.environ.get("MASTER_PORT", "29511"))
        _STORE = td.TCPStore(addr, port + 7, world, rank == 0,
                             timeout=datetime.timedelta(seconds=600))
    return _STORE


def exchange_uid(rank: int, world: int, tag: str = "uid") -> bytes | None:
    if world == 1:
        return None
    st = store(rank, world)
    key = f"hexexec/{tag}"
    if rank == 0:
        st.set(key, unique_id())
    return bytes(st.get(key))


def barrier(rank: int, world: int, tag: str):
    if world == 1:
        return
    st = store(rank, world)
    st.add(f"hexexec/bar/{tag}", 1)
    st.wait([f"hexexec/bar/{tag}"])
    while int(st.add(f"hexexec/bar/{tag}", 0)) < world:
        import time
        time.sleep(0.001)


def make_executor(cluster: str, model: str, plan: str, exec_config=None, tag="uid"):
    rank, world, local = env_rank()
    uid = exchange_uid(rank, world, tag)
    return Executor(cluster, model, plan, exec_config, rank=rank, world_size=world,
                    device=local, uid=uid)
