"""Build recipe for the nulpa CUDA library (sm_100a) and the test-only checkers.

    python -m paper_2411_11468_b200.build          # libnulpa.so (+ oracle/ checkers)

Outputs stay in-tree (git-ignored, shipped to the GPU box with the repo):
    paper_2411_11468_b200/libnulpa.so      C ABI + C++ drop-in (the product)
    build/nulpa_tests                      C++ drop-in KAT binary (tests/cpp)
    oracle/liboracle.so                    C restatement (test infrastructure)
    oracle/_ref/libnulpa_ref.so            reference library (only where /root/reference exists)
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libnulpa.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# tuning experiments: extra nvcc flags (e.g. -DNULPA_WIDE_LIMIT=8192); rebuild with force=True
EXTRA_NVCC = os.environ.get("NULPA_NVCC_FLAGS", "").split()
CU_SOURCES = ["graph.cu", "layout.cu", "engine.cu", "quality.cu", "gen.cu", "build_csr.cu", "textout.cu", "partition.cu"]
CXX_SOURCES = ["dropin.cpp", "textio.cpp"]


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} ... {cmd[-1]}")


def _newer(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return False
    t = target.stat().st_mtime
    return all(d.stat().st_mtime <= t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + list(
        (ROOT / "include").rglob("*.h*"))
    inc = ["-I", str(ROOT / "include"), "-I", str(CSRC)]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = CSRC / src
        o = OBJ / (src + ".o")
        objs.append(o)
        if force or not _newer(o, [s] + headers):
            jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                         "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr", *EXTRA_NVCC, *inc, "-c", str(s),
                         "-o", str(o)])
    for src in CXX_SOURCES:
        s = CSRC / src
        o = OBJ / (src + ".o")
        objs.append(o)
        if force or not _newer(o, [s] + headers):
            jobs.append(["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", *inc,
                         "-I", os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include"), "-c",
                         str(s), "-o", str(o)])
    if jobs:
        with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            list(ex.map(_run, jobs))
    if force or jobs or not LIB.exists():
        tmp = LIB.with_suffix(".so.tmp")
        _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)])
        os.replace(tmp, LIB)
    return LIB


def build_cpp_tests() -> Path:
    """C++ KAT binary for the drop-in (tests/cpp/test_dropin.cpp), linked to libnulpa.so."""
    out = ROOT / "build" / "nulpa_tests"
    src = ROOT / "tests" / "cpp" / "test_dropin.cpp"
    if not src.exists():
        return out
    deps = [src, LIB] + list((ROOT / "include").rglob("*.h*"))
    if not _newer(out, deps):
        out.parent.mkdir(parents=True, exist_ok=True)
        _run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), str(src), "-o", str(out),
              "-L", str(PKG), "-lnulpa", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../paper_2411_11468_b200"])
    return out


def build_tools() -> Path:
    """tools/cpp/dropin_e2e.cpp -> build/nulpa_dropin_e2e (bench.py's drop-in e2e leg)."""
    out = ROOT / "build" / "nulpa_dropin_e2e"
    src = ROOT / "tools" / "cpp" / "dropin_e2e.cpp"
    if not src.exists():
        return out
    deps = [src, LIB] + list((ROOT / "include").rglob("*.h*"))
    if not _newer(out, deps):
        out.parent.mkdir(parents=True, exist_ok=True)
        _run(["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), str(src), "-o", str(out),
              "-L", str(PKG), "-lnulpa", f"-Wl,-rpath,{PKG}",
              "-Wl,-rpath,$ORIGIN/../paper_2411_11468_b200"])
    return out


def build_checkers() -> None:
    """Test infrastructure only: oracle/liboracle.so and, where the reference
    sources exist, oracle/_ref/libnulpa_ref.so."""
    if shutil.which("make") is None:
        return
    _run(["make", "-s", "-C", str(ROOT / "oracle")])


def main() -> None:
    force = "--force" in sys.argv
    build_library(force=force)
    build_checkers()
    build_cpp_tests()
    build_tools()
    print(LIB)


if __name__ == "__main__":
    main()
