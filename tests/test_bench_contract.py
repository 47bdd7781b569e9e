"""bench.py's reference arm (CPU, no GPU needed): it times the unmodified
reference (oracle/_ref) and must not map the product library; its `config`
is the GPU arm's, so the driver can compare the two lines."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libablmc_ref.so"


@pytest.mark.skipif(not REF_SO.exists(), reason="oracle/_ref not built")
def test_reference_arm_never_loads_the_product_library():
    code = (
        "import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', "
        "'--warmup', '0', '--level', '4', '--ref-step-seconds', '0.2']\n"
        "runpy.run_path('bench.py', run_name='__main__')\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('MAPS_HAS_PRODUCT', 'libablmc_b200' in maps, 'MAPS_HAS_REF', 'libablmc_ref' in maps)\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "MAPS_HAS_PRODUCT False MAPS_HAS_REF True" in r.stdout
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    sys.path.insert(0, str(ROOT))
    import argparse

    import bench
    a = argparse.Namespace(level=4, integrator="se", paths=1 << 25)
    assert line["config"] == bench.workload_config(a, 1)  # the GPU arm's config
    assert "paths_per_step" in line["cpu_sample"]


@pytest.mark.skipif(not REF_SO.exists(), reason="oracle/_ref not built")
def test_gpus_n_spawns_its_own_ranks():
    """`bench.py --gpus 2` outside torchrun re-executes itself under
    torch.distributed.run (2 ranks); for the reference arm rank 0 alone runs
    and prints the one JSON line."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--level", "3",
                        "--ref-step-seconds", "0.2"], cwd=ROOT, capture_output=True, text=True,
                       timeout=300, env={**__import__("os").environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
    assert line["config"]["parallelism"].startswith("dp2")
