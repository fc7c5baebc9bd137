"""Worker for tests/test_dist_cpu.py, launched with torchrun (world size 2,
gloo, 127.0.0.1).  Exercises the host-side data-parallel logic of the
training step (§5.4): contiguous batch sharding, the rank-0
broadcast of an opaque 128-byte id (as bench.py does for ncclUniqueId), the
bucket plan every rank must agree on, gradient averaging by all-reduce, and
the max-over-ranks step time."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    out_dir = sys.argv[1]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    import synth
    from oracle import nets
    from oracle.step import train_step, _shard
    import paper_1912_01703_b200 as be

    # 1. opaque id broadcast (bench.py's ncclUniqueId path)
    uid = [bytes(range(128)) if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ok_uid = uid[0] == bytes(range(128))

    # 2. bucket plan identical on every rank
    net_p = be.nn.ResNet50()
    numels = [int(np.prod(s[1])) for s in net_p.param_specs()]
    plan = be.ddp_plan(numels, 25 << 20)
    plans = [None] * world
    dist.all_gather_object(plans, plan)
    same_plan = all(p == plans[0] for p in plans)

    # 3. data-parallel step: shard, local grads, all-reduce average, SGD
    net = nets.MLP((20, 16, 5))
    P = synth.make_params(net.param_specs(), 1)
    x = synth.normal((8, 20), 1, 1)
    y = synth.labels(8, 5, 1)
    local = train_step(net, P, _shard((x, y), rank, world), lr=0.0)
    g = {k: torch.from_numpy(v.copy()) for k, v in local["grads"].items()}
    for k in sorted(g):
        dist.all_reduce(g[k], op=dist.ReduceOp.SUM)
        g[k] /= world
    emu = train_step(net, P, (x, y), lr=0.1, replicas=world)
    glob = train_step(net, P, (x, y), lr=0.1, replicas=1)
    err_emu = max(float(np.max(np.abs(g[k].numpy() - emu["grads"][k]))) for k in g)
    err_glob = max(float(np.max(np.abs(g[k].numpy() - glob["grads"][k]))) for k in g)
    new = {k: P[k].astype(np.float64) - 0.1 * g[k].numpy() for k in g}
    params = [None] * world
    dist.all_gather_object(params, {k: v.tolist() for k, v in new.items()})
    replicas_equal = all(p == params[0] for p in params)

    # 4. max-over-ranks timing reduction
    t = torch.tensor([10.0 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)

    res = dict(rank=rank, world=world, ok_uid=ok_uid, same_plan=same_plan, n_buckets=len(plan[2]),
               err_emu=err_emu, err_glob=err_glob, replicas_equal=replicas_equal, tmax=float(t.item()))
    json.dump(res, open(os.path.join(out_dir, f"rank{rank}.json"), "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
