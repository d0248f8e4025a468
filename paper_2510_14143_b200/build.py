"""In-tree build of the CUDA library (sm_100a only).

    python -m paper_2510_14143_b200.build

produces paper_2510_14143_b200/lib/libvkrl.so from csrc/*.cu with
`nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo`.  The .so is
git-ignored but travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libvkrl.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
    "-I" + os.path.join(ROOT, "include"),
]


def _nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


CLI_SRC = os.path.join(PKG, "host", "vk_cli.cu")
CLI = os.path.join(LIBDIR, "voxelkit_b200")


# rl_fast_len.cu is compiled once per compile-time FFT length (-DVK_LEN=N),
# the lengths listed in csrc/fast_lengths.def
def _fast_lengths():
    import re
    with open(os.path.join(CSRC, "fast_lengths.def")) as f:
        return tuple(int(m) for m in re.findall(r"^VK_FAST_LEN\((\d+)\)", f.read(), re.M))


FAST_LENGTHS = _fast_lengths()


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cpp")) and f != "rl_fast_len.cu")


def units(lengths=FAST_LENGTHS):
    """(source, extra flags, object name) for every object of the library."""
    u = [(src, [], os.path.splitext(os.path.basename(src))[0] + ".o") for src in sources()]
    u += [(os.path.join(CSRC, "rl_fast_len.cu"), [f"-DVK_LEN={n}"], f"rl_fast_len_{n}.o") for n in lengths]
    return u


def deps():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)) + [
        os.path.join(ROOT, "include", h) for h in ("vk_rl.h", "vk_io.h")]


def up_to_date() -> bool:
    if not (os.path.exists(LIB) and os.path.exists(CLI)):
        return False
    t = min(os.path.getmtime(LIB), os.path.getmtime(CLI))
    return all(os.path.getmtime(d) <= t for d in deps() + [CLI_SRC])


def build_cli(verbose: bool = False) -> str:
    """voxelkit_b200 (the CLI `deconvolve` on the B200 path), linked against
    lib/libvkrl.so with an $ORIGIN rpath."""
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
           "-I" + os.path.join(ROOT, "include"), "-o", CLI + ".tmp", CLI_SRC,
           "-L" + LIBDIR, "-lvkrl", "-Xlinker", "-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc (cli) failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    os.replace(CLI + ".tmp", CLI)
    return CLI


def build(force: bool = False, verbose: bool = False, variant: str = "", extra_flags=(), lengths=None) -> str:
    """variant: a side build (lib/<variant>/libvkrl.so, own objects) with
    extra_flags, for A/B measurements (load it with VK_RL_LIB=...); lengths:
    only these compile-time lengths (the others take the generic kernels),
    which keeps side libraries small enough for the size-capped snapshot."""
    lib = os.path.join(LIBDIR, variant, "libvkrl.so") if variant else LIB
    if not variant and not force and up_to_date():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    # side builds keep their objects out of the tree (the GPU snapshot is size-capped)
    objdir = os.path.join("/tmp", "vk_build_obj_" + variant) if variant else os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + list(extra_flags)
    if lengths:
        assert variant, "a length subset is for side builds only"
        deff = os.path.join(objdir, "fast_lengths.def")
        with open(deff, "w") as f:
            f.writelines(f"VK_FAST_LEN({n})\n" for n in lengths)
        compile_flags.append(f'-DVK_FAST_LENGTHS_DEF="{deff}"')
    lens = tuple(lengths) if lengths else FAST_LENGTHS

    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".def"))] + [
        os.path.join(ROOT, "include", h) for h in ("vk_rl.h", "vk_io.h")]
    newest_header = max(os.path.getmtime(h) for h in headers)

    def compile_one(unit):
        src, extra, obj = unit
        out = os.path.join(objdir, obj)
        if (not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src)
                and os.path.getmtime(out) >= newest_header and not extra_flags):
            return None, None  # up to date (source and every header older than the object)
        cmd = [_nvcc(), *compile_flags, *extra, "-c", "-o", out, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    from concurrent.futures import ThreadPoolExecutor

    # the per-length kernels dominate the build: compile every object at once
    with ThreadPoolExecutor(max_workers=max(1, os.cpu_count() or 1)) as ex:
        results = list(ex.map(compile_one, units(lens)))
    for cmd, r in results:
        if cmd is None:
            continue
        if verbose:
            print(" ".join(cmd))
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr)
    tmp = lib + ".tmp"
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
           *[os.path.join(objdir, u[2]) for u in units(lens)]]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc (link) failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    if variant:
        return lib
    build_cli(verbose)
    return LIB


if __name__ == "__main__":
    if "--variant" in sys.argv:  # python -m paper_2510_14143_b200.build --variant NAME -DFLAG=1 ...
        i = sys.argv.index("--variant")
        rest = sys.argv[i + 2:]
        lens = None
        if "--lengths" in rest:  # --lengths 2160,1080
            j = rest.index("--lengths")
            lens = [int(n) for n in rest[j + 1].split(",")]
            rest = rest[:j] + rest[j + 2:]
        print(build(verbose=False, variant=sys.argv[i + 1], extra_flags=rest, lengths=lens))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
