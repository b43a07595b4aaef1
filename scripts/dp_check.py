"""Multi-GPU parity (run under torchrun, >=2 GPUs): the NCCL-allreduced
gradient of groups sharded over ranks equals the single-device accumulation
of the same groups; the allreduced loss scalars equal their sum."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch.distributed as dist
from paper_2511_18871_b200 import parl as P
from paper_2511_18871_b200.dp import bootstrap_comm, rank_groups

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
dist.init_process_group("gloo")
ctx = P.Context(local, P.PREC_FP32)
bootstrap_comm(ctx, rank, world)
cfg = P.ModelConfig(4096, 256, 2, 4, 1024, 576)
tm = P.TriModel.init(cfg, 7, ctx)
tm.old_policy = tm.policy.clone(seed=3, noise=0.01)
rng = np.random.default_rng(5)
groups = [(rng.integers(4, 4096, 64), [rng.integers(4, 4096, n) for n in (100, 130, 90, 128)], rng.random(4))
          for _ in range(2 * world)]
hyper = P.HyperParams()
grads = P.GradBuffer(tm.policy)
grp = P.Group(576, 4, ctx)
ctx.stats_reset()
for gi in rank_groups(len(groups), None, world, rank):
    pr, rs, rw = groups[gi]
    grp.pack(pr, rs, 576)
    P.train_microbatch(tm, grp, grads, hyper, rewards=rw, want_stats=False)
grads.allreduce()
ctx.stats_allreduce()
g_dp, st_dp = grads.flat(), ctx.stats()
# the same step with the allreduce overlapped with the last micro-batch's backward
grads.reset()
mine = list(rank_groups(len(groups), None, world, rank))
for n_, gi in enumerate(mine):
    pr, rs, rw = groups[gi]
    grp.pack(pr, rs, 576)
    if n_ == len(mine) - 1:
        grads.allreduce_overlap()
    P.train_microbatch(tm, grp, grads, hyper, rewards=rw, want_stats=False)
grads.allreduce()
g_ov = grads.flat()
rel_ov = np.linalg.norm(g_ov - g_dp) / np.linalg.norm(g_dp)
print(f"DP_CHECK rank={rank} overlapped vs whole-buffer allreduce rel={rel_ov:.3e}")
assert rel_ov < 1e-6, "overlapped allreduce differs"  # (PARL_AR_OVERLAP=1 arms the streaming path)
if rank == 0:
    ctx1 = P.Context(local, P.PREC_FP32)
    tm1 = P.TriModel(P.ModelParams.from_flat(cfg, tm.policy.flat(), ctx=ctx1),
                     P.ModelParams.from_flat(cfg, tm.old_policy.flat(), ctx=ctx1),
                     P.ModelParams.from_flat(cfg, tm.reference.flat(), ctx=ctx1))
    g1 = P.GradBuffer(tm1.policy)
    grp1 = P.Group(576, 4, ctx1)
    ctx1.stats_reset()
    for pr, rs, rw in groups:
        grp1.pack(pr, rs, 576)
        P.train_microbatch(tm1, grp1, g1, hyper, rewards=rw, want_stats=False)
    g_ref, st_ref = g1.flat(), ctx1.stats()
    rel = np.linalg.norm(g_dp - g_ref) / np.linalg.norm(g_ref)
    obj = abs(st_dp["objective_sum"] - st_ref["objective_sum"])
    print(f"DP_CHECK world={world} grad_rel={rel:.3e} obj_diff={obj:.3e} units={st_dp['total_units']}/{st_ref['total_units']}")
    assert rel < 1e-5 and obj < 1e-6 and st_dp["total_units"] == st_ref["total_units"], "dp parity failed"
    print("DP_CHECK OK")
dist.barrier()
dist.destroy_process_group()
