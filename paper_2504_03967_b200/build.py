"""In-tree build of libqgear_b200.so (nvcc, sm_100a).  `python -m paper_2504_03967_b200.build`"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libqgear_b200.so")
BUILD = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
SOURCES = ["plan.cpp", "container.cpp", "capi.cu", "fused.cu", "reduce.cu", "ucry.cu", "tree.cu", "jit.cpp"]
HEADERS = ["desc.h", "kernels.h", "plan.h", "jt_lists.h", "jit.h"]


def jump_table_ok(ptx: str) -> bool:
    """fused.cu's run_op enters its switch through a PTX jump table whose targets
    are inline-asm labels (QGJ_*).  Jumping to a label skips whatever NVVM placed
    before it in the same basic block, so every label must directly follow a
    block label or a branch."""
    lines = ptx.split("\n")
    n = 0
    for i, line in enumerate(lines):
        if not re.match(r"\s*QGJ_\w+:\s*$", line):
            continue
        n += 1
        j = i - 1
        while j >= 0 and (not lines[j].strip() or lines[j].strip().startswith(("//", ".loc"))):
            j -= 1
        prev = lines[j].strip() if j >= 0 else ""
        if not (re.match(r"^\$L__BB\w+:$", prev) or re.match(r"^(@!?%p\d+ )?bra(\.uni)?\s", prev)):
            return False
    return n > 0 and ptx.count("brx.idx") > 0


def _newest_input() -> float:
    paths = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    paths.append(os.path.join(ROOT, "include", "qgear_b200.h"))
    paths.append(os.path.abspath(__file__))
    return max(os.path.getmtime(p) for p in paths)


def _deps(path: str, seen=None) -> list:
    """path + every local header it includes (recursively, quoted includes only)."""
    seen = [] if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.append(path)
    for line in open(path, errors="replace"):
        m = re.match(r'\s*#\s*include\s+"([^"]+)"', line)
        if m:
            _deps(os.path.normpath(os.path.join(os.path.dirname(path), m.group(1))), seen)
    return seen


def _compile(src: str, force: bool = True) -> str:
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    if not force and os.path.exists(obj):  # incremental: the source's own #include closure
        deps = _deps(os.path.join(CSRC, src)) + [os.path.abspath(__file__)]
        if os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
            return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-warn-spills"]
    keep = os.path.join(BUILD, "keep_" + os.path.splitext(src)[0])
    if src == "fused.cu":  # keep the PTX of this very compilation for the jump-table check
        os.makedirs(keep, exist_ok=True)
        cmd += ["-keep", "-keep-dir", keep]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if src == "fused.cu":
        ptx = os.path.join(keep, "fused.ptx")
        if not os.path.exists(ptx) or not jump_table_ok(open(ptx).read()):
            sys.stderr.write("fused.cu: PTX jump-table check failed; building the compare-tree dispatch\n")
            r = subprocess.run(cmd + ["-DQG_NO_JT"], capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build_counts_ext(force: bool = False) -> str:
    """The host-side CPython helper `_counts` (csrc/counts_dict.c: the {bitstring: count} dict)."""
    import sysconfig

    src = os.path.join(CSRC, "counts_dict.c")
    out = os.path.join(PKG, "_counts" + sysconfig.get_config_var("EXT_SUFFIX"))
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
        return out
    cmd = ["gcc", "-O2", "-shared", "-fPIC", "-Wall", f"-I{sysconfig.get_paths()['include']}", src, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"gcc failed for counts_dict.c:\n{r.stdout}\n{r.stderr}")
    return out


def build(force: bool = False, verbose: bool = True) -> str:
    build_counts_ext(force)
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= _newest_input():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda src: _compile(src, force), SOURCES))
    cmd = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-cudart", "static",
           "-L/usr/local/cuda/lib64", "-lnvptxcompiler_static", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
