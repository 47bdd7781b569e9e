"""Run under torch.distributed.run (NCCL, one process per GPU): the sharded
accumulate (super-block partials + one all-gather + ordered merge) must give
the same bits on every rank as a single-process accumulate_samples."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_07717_b200 import ablmc  # noqa: E402
from paper_1612_07717_b200.sharding import accumulate_sharded  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ablmc.init(local)
    pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.gl, ablmc.QoISpec(), 0.05, 0.1,
                            1.0, 2, 21)
    count = 3 * (1 << 22) + 777
    acc = ablmc.LevelStats().init(2, pr.h_level(2), 1)
    accumulate_sharded(acc, 5, count, pr, 2)
    one = ablmc.LevelStats().init(2, pr.h_level(2), 1)
    ablmc.accumulate_samples(one, 5, count, pr, 2)
    ok = (acc.sum_y[0] == one.sum_y[0] and acc.sum_y2[0] == one.sum_y2[0] and acc.n == one.n
          and acc.cost_steps == one.cost_steps)
    print(f"rank {dist.get_rank()}/{dist.get_world_size()} sharded == single: {ok} "
          f"({acc.sum_y[0]!r} vs {one.sum_y[0]!r})", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
