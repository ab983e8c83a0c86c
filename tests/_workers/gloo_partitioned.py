"""Worker for tests/test_multigpu_gloo.py: one rank of the tree-partitioned
protocol on the CPU oracle (TEST INFRASTRUCTURE).  Each rank computes only the
agents tree_placement gives it and hands every chunk's tokens / logprobs /
entropies from the owner to the other ranks -- the message pattern the C++
engine issues over NCCL P2P (csrc/host/engine.cpp phase A)."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from oracle.configs import models_of, run_config  # noqa: E402
from oracle.orchestrator import run_query  # noqa: E402


def main():
    cfg = json.loads(sys.argv[1])
    sample, out = int(sys.argv[2]), sys.argv[3]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    sent = [0]

    def exchange(rid, owner, n, payload):
        if rank == owner:
            t = (torch.tensor(payload[0], dtype=torch.int64), torch.tensor(payload[1], dtype=torch.float64),
                 torch.tensor(payload[2], dtype=torch.float64))
            for peer in range(world):
                if peer != rank:
                    for x in t:
                        dist.send(x, peer)
            sent[0] += n
            return payload
        t = (torch.empty(n, dtype=torch.int64), torch.empty(n, dtype=torch.float64), torch.empty(n, dtype=torch.float64))
        for x in t:
            dist.recv(x, owner)
        return t[0].tolist(), t[1].tolist(), t[2].tolist()

    forced = None
    if len(sys.argv) > 4:  # replay: this rank's own agents only, the rest must arrive by exchange
        with open(sys.argv[4]) as f:
            forced = {tuple(int(x) for x in k.split(":")): tuple(v) for k, v in json.load(f)[rank].items()}
    models = {} if forced is not None else models_of(cfg, 512)
    o = run_query(run_config(cfg), models, sample, forced=forced, world=world, rank=rank, exchange=exchange)
    o.pop("events")
    o["sent_tokens"] = sent[0]
    with open(out, "w") as f:
        json.dump(o, f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
