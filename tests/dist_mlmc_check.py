"""Run under torch.distributed.run with any world size: the host MLMC driver
(run_mlmc) and accumulate_samples with the library's collective enabled must
give, on every rank, exactly the bits of the single-process run.

Backend: NCCL when every rank has its own GPU; otherwise gloo, so several
ranks may share one GPU (their kernels never wait on each other: the exchange
is a host-side all-gather between accumulate calls)."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_07717_b200 import ablmc  # noqa: E402
from paper_1612_07717_b200.sharding import disable_collective, enable_collective  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    ngpu = torch.cuda.device_count()
    dev = local % ngpu
    torch.cuda.set_device(dev)
    backend = "nccl" if world <= ngpu else "gloo"
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo")
    ablmc.init(dev)
    pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.gl, ablmc.QoISpec(), 0.05, 0.1,
                            1.0, 40, 555)
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(8, 1.0))
    prb = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, q, 0.05, 0.1, 1.0, 4, 9)
    count = 5 * (1 << 22) + 4321

    def run():
        a = ablmc.LevelStats().init(3, prb.h_level(3), prb.dim())
        ablmc.accumulate_samples(a, 11, count, prb, 3)
        m = ablmc.run_mlmc(pr, 1e-3)
        js = ablmc.result_json(ablmc.RunConfig(timings=False), m)  # byte-stable result.json
        return (a.sum_y.tobytes(), a.sum_y2.tobytes(), a.n, a.cost_steps, m.estimate, m.stat_error,
                [(s.n, s.sum_y.tobytes(), s.sum_y2.tobytes()) for s in m.level_stats], js)

    single = run()
    enable_collective()
    shared = run()
    # one allocation round of four levels: ONE all-gather
    from paper_1612_07717_b200 import sharding
    c0 = sharding.collective_calls
    reqs = [(ablmc.LevelStats().init(l, pr.h_level(l), 1), 0, 1000 << (4 - l), l) for l in range(4)]
    ablmc.accumulate_levels(reqs, pr)
    one_per_round = sharding.collective_calls - c0 == 1 and ablmc.last_collective_count() == 1
    disable_collective()
    ok = single == shared and one_per_round
    print(f"rank {dist.get_rank()}/{world} ({backend}) collective == single-process: {ok}",
          flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
