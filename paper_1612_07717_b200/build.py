"""In-tree build of the product library ``libablmc_b200.so`` (sm_100a only).

nvcc cross-compiles here without a GPU; the ``.so`` is git-ignored but travels
to the GPU box with the repo snapshot.  Usage: ``python -m paper_1612_07717_b200.build``.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "libablmc_b200.so"
SOURCES = ["level_kernels.cu", "adaptive_kernels.cu", "binned_kernels.cu", "collective.cu", "capi.cu", "drivers.cu",
           "output.cpp"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -ffp-contract=off for host code: host_coeffs (capi.cu) must round like the
# device's IEEE path
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "-I",
         str(ROOT / "include")]
# nlohmann/json (header-only, shipped in this image under cudnn_frontend) for
# byte-identical result.json output (csrc/output.cpp).
NLOHMANN = Path(os.environ.get(
    "ABLMC_NLOHMANN_DIR",
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"))
CXXFLAGS = ["-std=c++17", "-O2", "-fPIC", "-Wall", "-Wextra", "-I", str(ROOT / "include"),
            "-I", str(NLOHMANN)]


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    headers = list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "ablmc_b200.h"]
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = OBJ / (s.stem + ".o")
        if force or _stale(o, [s, *headers]):
            if s.suffix == ".cpp":
                cmd = [CXX, *CXXFLAGS, "-c", str(s), "-o", str(o)]
            else:
                cmd = [NVCC, *ARCH, *FLAGS, "-c", str(s), "-o", str(o)]
            if src.endswith("_kernels.cu"):
                cmd += ["-Xptxas", "-v"]
            jobs.append((cmd, o))

    def run(job):
        cmd, o = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {o.name}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            (OBJ / (o.stem + ".ptxas.txt")).write_text(r.stderr)
        return o

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    objs = [OBJ / (Path(s).stem + ".o") for s in SOURCES]
    if force or jobs or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def build_oracle() -> None:
    """Compile the parity checkers (oracle/), test infrastructure only."""
    r = subprocess.run(["make", "-s", "-f", str(ROOT / "oracle" / "Makefile")], capture_output=True,
                       text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


REF_INCLUDE = Path("/root/reference/proj/include")
DEMO = ROOT / "integration" / "adapter_demo"


def build_integration_demo() -> None:
    """integration/adapter_demo: the reference's own code calling this library
    through integration/ablmc_b200_adapter.hpp (needs the reference headers,
    so it is built here only; the binary travels to the GPU box)."""
    if not REF_INCLUDE.is_dir():
        return
    src = ROOT / "integration" / "adapter_demo.cpp"
    deps = [src, ROOT / "integration" / "ablmc_b200_adapter.hpp", LIB]
    if not _stale(DEMO, deps):
        return
    cmd = ["g++", "-std=gnu++20", "-O2", "-pthread", f"-I{REF_INCLUDE}", f"-I{ROOT / 'include'}",
           f"-I{ROOT / 'integration'}", str(src), "-o", str(DEMO), f"-L{PKG}", "-l:libablmc_b200.so",
           "-Wl,-rpath,$ORIGIN/../paper_1612_07717_b200"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"adapter demo build failed:\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    lib = build(verbose=True, force="--force" in sys.argv)
    build_oracle()
    build_integration_demo()
    print(lib)
