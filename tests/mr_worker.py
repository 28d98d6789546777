"""One CPU rank of tests/test_multirank_cpu.py (gloo, no GPU): the host side
of the N > 1 path -- NCCL-id exchange through the TCPStore, per-rank
validate_only executors (layout + arena sizing), and the cross-rank
invariants NCCL relies on, checked with torch.distributed (gloo)."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch.distributed as td

    import bench
    from paper_2409_01143_b200 import dist
    from paper_2409_01143_b200.hexexec import Executor, Plan
    plans = sys.argv[1].split(",")
    rank, world, _ = dist.env_rank()
    td.init_process_group("gloo", rank=rank, world_size=world)
    out = {"rank": rank}
    # NCCL unique id created on rank 0, shared through the store
    try:
        uid = dist.exchange_uid(rank, world, "uid-cpu")
        out["uid_len"] = len(uid)
        h = hashlib.sha256(uid).hexdigest()
        allh = [None] * world
        td.all_gather_object(allh, h)
        out["uid_same"] = len(set(allh)) == 1
    except Exception as e:  # noqa: BLE001
        out["uid_error"] = str(e)[:200]
    for name in plans:
        c, m, p, _ = bench.load(name)
        pl = Plan(c, m, p)
        lay = pl.layout()
        if pl.world_size != world:
            continue
        ex = Executor(c, m, p, {"validate_only": True}, rank=rank, world_size=world)
        st = ex.stats()
        ex.close()
        mine = lay["ranks"][rank]
        # every rank derives the same layout from the same documents
        digest = hashlib.sha256(json.dumps(lay, sort_keys=True).encode()).hexdigest()
        alld = [None] * world
        td.all_gather_object(alld, digest)
        # per communicator: the DP bucket sequence (group, count) of every member
        # must be identical, or the grouped ncclAllReduce calls would not match
        seqs = {}
        for b in mine.get("dp_buckets", []):
            seqs.setdefault(str(b["comm"]), []).append([b["group"], b["count"]])
        alls = [None] * world
        td.all_gather_object(alls, seqs)
        agree = all(seqs[cm] == s2[cm] for s2 in alls for cm in s2 if cm in seqs)
        # every communicator a rank joins is joined by exactly its member set
        members = {str(i): set(cs) for i, cs in enumerate(lay["comm_sets"])}
        joined = all(rank in members[cm] for cm in seqs)
        # PP peers are symmetric: each rank I send activations to receives them from me
        peers = [None] * world
        td.all_gather_object(peers, mine.get("fwd_recv_from", -1))
        sym = all(peers[q] == rank for q in mine.get("fwd_send_to", []))
        mx = bench.gather_max([float(st["arena_bytes"])], rank, world, f"mx-{name}")[0]
        out[name] = {"layout_same": len(set(alld)) == 1, "bucket_seq_agree": agree and joined,
                     "pp_symmetric": sym, "arena_bytes": st["arena_bytes"], "arena_max": mx,
                     "active": st["active"], "buckets": sum(len(v) for v in seqs.values())}
    dist.barrier(rank, world, "end")
    td.destroy_process_group()
    print("MR " + json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
