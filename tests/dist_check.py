"""Run under torch.distributed.run (one process per GPU): the library's
NATIVE NCCL group (ablmc_init_group; the unique id travels over
torch.distributed, the data path is the library's own all-gather on its
stream) must give, on every rank, exactly the bits of the single-process
calls -- accumulate_samples, one accumulate_levels batch (ONE all-gather for
all its levels), run_mlmc and the device-resident accumulate."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_07717_b200 import ablmc  # noqa: E402
from paper_1612_07717_b200.sharding import init_nccl_group  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ablmc.init(local)
    pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.gl, ablmc.QoISpec(), 0.05, 0.1,
                            1.0, 2, 21)
    count = 3 * (1 << 22) + 777

    def run():
        out = []
        a = ablmc.LevelStats().init(2, pr.h_level(2), 1)
        ablmc.accumulate_samples(a, 5, count, pr, 2)
        out.append((a.sum_y.tobytes(), a.sum_y2.tobytes(), a.n, a.cost_steps))
        reqs = [(ablmc.LevelStats().init(l, pr.h_level(l), 1), 3 * l, count >> l, l)
                for l in range(4)]
        ablmc.accumulate_levels(reqs, pr)
        out.append(ablmc.last_collective_count())
        out += [(r[0].sum_y.tobytes(), r[0].sum_y2.tobytes(), r[0].n) for r in reqs]
        m = ablmc.run_mlmc(pr, 1e-3)
        out.append((m.estimate, m.stat_error, [(s.n, s.sum_y.tobytes()) for s in m.level_stats]))
        lib = ablmc.lib()
        import ctypes as C
        ablmc._check(lib.ablmc_accumulate_device(C.byref(pr._c), 3, 0, count))
        d = ablmc.LevelStats().init(3, pr.h_level(3), 1)
        v = d._view()
        ablmc._check(lib.ablmc_fetch_device_result(C.byref(pr._c), 3, C.byref(v)))
        d._take(v)
        out.append((d.sum_y.tobytes(), d.n, d.cost_steps))
        return out

    single = run()
    assert single[1] == 0  # no collective in single-device mode
    init_nccl_group()
    info = ablmc.group_info()
    shared = run()
    ok = (info["mode"] == 2 and info["world"] == dist.get_world_size() and shared[1] == 1
          and single[:1] + single[2:] == shared[:1] + shared[2:])
    print(f"rank {dist.get_rank()}/{dist.get_world_size()} native group {info}: "
          f"sharded == single: {ok}", flush=True)
    ablmc.init(local)  # back to single-device mode (destroys the communicator)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
