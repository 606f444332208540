"""Build every native artefact in-tree (called by __graft_entry__.build()).

  inputs/libcbp_inputs.so            seeded QC constructor (shared input generator)
  oracle/liboracle.so                CPU oracle (test infrastructure; g++ -ffp-contract=off)
  paper_2305_05286_b200/libcbp.so    the product: C-ABI host code + sm_100a kernels

Rebuilds a target only when one of its sources (or this file) is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# arithmetic contract: no implicit FMA contraction, IEEE div/sqrt, denormals kept
NVCC_CONTRACT = ["--fmad=false", "--prec-div=true", "--prec-sqrt=true", "--ftz=false"]

INPUTS_SRC = [ROOT / "inputs" / "qc_construct.c"]
ORACLE_SRC = [ROOT / "oracle" / "cbp_oracle.cpp", ROOT / "oracle" / "contract32.c"]
CBP_SRC = sorted((ROOT / "paper_2305_05286_b200" / "csrc").glob("*.cu")) + sorted(
    (ROOT / "paper_2305_05286_b200" / "csrc").glob("*.cpp"))
# every file under csrc/ (kernels, host code, *.cuh and *.h headers) is a dependency of libcbp.so
CBP_HDR = sorted(p for p in (ROOT / "paper_2305_05286_b200" / "csrc").iterdir() if p.is_file()) + [
    ROOT / "include" / "cbp.h", ROOT / "inputs" / "cbp_inputs.h"]

INPUTS_SO = ROOT / "inputs" / "libcbp_inputs.so"
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
CBP_SO = ROOT / "paper_2305_05286_b200" / "libcbp.so"


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in list(deps) + [Path(__file__)])


def _run(cmd, cwd=ROOT):
    print("+", " ".join(str(c) for c in cmd), flush=True)
    subprocess.run([str(c) for c in cmd], check=True, cwd=cwd)


def build_inputs(force=False):
    if force or _stale(INPUTS_SO, INPUTS_SRC + [ROOT / "inputs" / "cbp_inputs.h"]):
        _run(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", *INPUTS_SRC, "-o", INPUTS_SO])
    return INPUTS_SO


def build_oracle(force=False):
    deps = ORACLE_SRC + INPUTS_SRC + [ROOT / "oracle" / "cbp_oracle.h", ROOT / "oracle" / "contract32.h"]
    if force or _stale(ORACLE_SO, deps):
        objs = []
        tmp = ROOT / "build" / "oracle"
        tmp.mkdir(parents=True, exist_ok=True)
        for src in ORACLE_SRC + INPUTS_SRC:
            obj = tmp / (src.stem + ".o")
            if src.suffix == ".c":
                cmd = ["gcc", "-std=c11"]
            else:
                cmd = ["g++", "-std=c++17"]
            _run(cmd + ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-Wall", "-Wextra",
                        "-I", ROOT / "oracle", "-I", ROOT / "inputs", "-c", src, "-o", obj])
            objs.append(obj)
        _run(["g++", "-shared", *objs, "-o", ORACLE_SO, "-lm"])
    return ORACLE_SO


def build_cbp(force=False, out=None, defines=()):
    """libcbp.so; `out`/`defines` build an alternate variant (kernel A/B experiments,
    loaded with CBP_LIB=<path>)."""
    out = Path(out) if out else CBP_SO
    deps = CBP_SRC + CBP_HDR + INPUTS_SRC
    if force or _stale(out, deps):
        tmp = ROOT / "build" / ("cbp" if out == CBP_SO else "cbp_" + out.stem)
        tmp.mkdir(parents=True, exist_ok=True)
        common = ["-I", ROOT / "include", "-I", ROOT / "inputs", "-I", ROOT / "paper_2305_05286_b200" / "csrc"]
        cmds = [[NVCC, "-std=c++17", *ARCH, "-O3", "-lineinfo", *NVCC_CONTRACT, "-Xptxas", "-v",
                 "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-Xcompiler", "-ffp-contract=off",
                 *[f"-D{d}" for d in defines], *common, "-c", src, "-o", tmp / (src.stem + ".o")] for src in CBP_SRC]
        objs = [c[-1] for c in cmds]
        # one nvcc per translation unit, in parallel (the kernels are split by algorithm)
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
            list(ex.map(_run, cmds))
        inp_obj = tmp / "qc_construct.o"
        _run(["gcc", "-std=c11", "-O2", "-fPIC", "-c", INPUTS_SRC[0], "-o", inp_obj])
        objs.append(inp_obj)
        _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *objs, "-o", out])
    return out


def build_all(force=False):
    build_inputs(force)
    build_oracle(force)
    if CBP_SRC:
        build_cbp(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
