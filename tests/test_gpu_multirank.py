"""Multi-rank member sharding on the GPU: two
ranks, each owning half of the members (strong scaling of the fixed member
set), exchanging only the sketch rows (one all-reduce), must give every
member the SAME increment and traces, bit for bit, as the single-rank pass.

Both ranks run on cuda:0 with gloo collectives (the box has one GPU); their
kernels never wait on each other -- the only exchange is the host-mediated
all-reduce of Gamma before the Nystrom stage (parallel.gather_sketch_rows).
"""

import os
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rank_pass(rank, world, port, cfg_id, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2605_23571_b200 import build
    build.build()
    from paper_2605_23571_b200.engine import EdaPass
    from paper_2605_23571_b200.parallel import shard
    from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble
    cfg = BASELINE_CONFIGS[cfg_id]
    offset, count = shard(cfg.members, world, rank)
    dens = build_ensemble(cfg, members=count, member_offset=offset)
    eng = EdaPass(dens, member_offset=offset, total_members=cfg.members, distributed=True)
    res = eng.run()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), offset=offset, x=res.x.cpu().numpy(),
             cost=np.array([t.cost for t in res.traces]),
             resnorm=np.array([t.resnorm for t in res.traces]),
             gamma=res.gamma.cpu().numpy(), values=res.approx.values)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg_id", [3, 4])
def test_two_rank_sharded_pass_is_bit_identical(cfg_id):
    import torch.multiprocessing as mp
    from paper_2605_23571_b200 import build
    build.build()
    from paper_2605_23571_b200.engine import EdaPass
    from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble
    cfg = BASELINE_CONFIGS[cfg_id]
    ref = EdaPass(build_ensemble(cfg)).run()
    X = ref.x.cpu().numpy()
    with tempfile.TemporaryDirectory() as d:
        port = 29600 + (os.getpid() % 500) + cfg_id
        mp.spawn(_rank_pass, args=(2, port, cfg_id, d), nprocs=2, join=True)
        parts = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(2)]
    covered = 0
    for p in parts:
        off, m = int(p["offset"]), p["x"].shape[0]
        np.testing.assert_array_equal(p["gamma"], ref.gamma.cpu().numpy())
        np.testing.assert_array_equal(p["values"], ref.approx.values)
        np.testing.assert_array_equal(p["x"], X[off:off + m])
        np.testing.assert_array_equal(p["cost"], np.array([t.cost for t in ref.traces[off:off + m]]))
        np.testing.assert_array_equal(p["resnorm"],
                                      np.array([t.resnorm for t in ref.traces[off:off + m]]))
        covered += m
    assert covered == cfg.members
