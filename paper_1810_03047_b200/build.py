"""Build libqtm.so (sm_100a) in-tree with nvcc.

Each trajectory-kernel variant is instantiated in its own translation unit
(csrc/gen/variant_<i>.cu) so the instantiations compile in parallel; the
C-ABI (csrc/qtm_capi.cu) includes the generated table.

    python -m paper_1810_03047_b200.build [--force] [--jobs N]
"""

from __future__ import annotations

import argparse
import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
GEN = os.path.join(CSRC, "gen")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libqtm.so")
# The throughput build contracts a*b+c into fused multiply-adds (rounding then
# differs from the reference's unfused numba arithmetic by ~1 ulp per op, the
# same order as the tree reductions; the whole GPU suite, reference-scale
# parity included, is green with it).  QTM_FMAD=0 builds the unfused parity
# library (every flop one DMUL/DADD, as numba); QTM_BUILD_TAG / QTM_LIB select
# an alternative library file for A/B runs.
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FMAD = os.environ.get("QTM_FMAD", "1") == "1"
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", f"-fmad={'true' if FMAD else 'false'}",
                     f"-DQTM_FMAD={1 if FMAD else 0}", "-Xcompiler", "-fPIC", "-I", INCLUDE]
# extra nvcc flags for A/B experiments (e.g. -DQTM_SPMV_PF(E)=0)
NVCC_FLAGS = NVCC_FLAGS + os.environ.get("QTM_NVCC_EXTRA", "").split()
if os.environ.get("QTM_PHASES", "0") == "1":
    NVCC_FLAGS = NVCC_FLAGS + ["-DQTM_PHASES"]
_TAG = os.environ.get("QTM_BUILD_TAG", "")
if _TAG:
    LIB = os.path.join(HERE, f"libqtm_{_TAG}.so")
    OBJ = os.path.join(HERE, f"_build_{_TAG}")

# (threads per CTA, components per thread, register-resident Nordsieck rows,
#  min CTAs per SM for __launch_bounds__, auto-select for dim <= this (0 = never)
#  [, time-dependent generator terms compiled in])
VARIANTS = [
    (32, 1, 13, 16, 0),      # 0
    (64, 1, 13, 8, 64),      # 1
    (96, 1, 13, 5, 0),       # 2
    (128, 1, 13, 4, 128),    # 3
    (256, 1, 13, 2, 256),    # 4
    (512, 1, 10, 1, 512),    # 5
    (512, 2, 8, 1, 0),       # 6  (the automatic choice up to d = 1024 before #22)
    (1024, 1, 6, 1, 0),      # 7
    (512, 2, 5, 1, 0),       # 8
    (1024, 2, 4, 1, 2048),   # 9
    # exploration: lower register caps / more CTAs per SM
    (32, 1, 9, 24, 0),       # 10
    (32, 1, 9, 32, 0),       # 11
    (96, 1, 9, 8, 96),       # 12
    (128, 1, 9, 6, 0),       # 13
    (256, 4, 5, 2, 0),       # 14
    (256, 4, 4, 2, 0),       # 15
    (512, 2, 4, 2, 0),       # 16
    # history in shared memory (RREG = 0): compact code, few registers
    (32, 1, 0, 24, 32),      # 17
    (64, 1, 0, 12, 0),       # 18
    (96, 1, 0, 8, 0),        # 19
    (128, 1, 0, 6, 0),       # 20
    (32, 1, 0, 32, 0),       # 21
    # one CTA per SM with fewer, wider threads: up to 255 registers each
    (256, 4, 8, 1, 0),       # 22 (automatic for 512 < d <= 1024 before #39: c4 1.44x, c5 1.19x faster than #6)
    (256, 4, 10, 1, 0),      # 23
    (256, 4, 6, 1, 0),       # 24
    (128, 8, 5, 1, 0),       # 25
    # two CTAs per SM with fewer, wider threads (d ~ 900, low order)
    (128, 8, 4, 2, 0),       # 26
    (192, 5, 4, 2, 0),       # 27
    # time-dependent H(t) (timedep.py): the automatic chain again, with the
    # G_k terms compiled in (selected only for problems with n_td > 0)
    (32, 1, 0, 24, 32, True),      # 28
    (64, 1, 13, 8, 64, True),      # 29
    (96, 1, 9, 8, 96, True),       # 30
    (128, 1, 13, 4, 128, True),    # 31
    (256, 1, 13, 2, 256, True),    # 32
    (512, 1, 10, 1, 512, True),    # 33
    (512, 2, 8, 1, 0, True),       # 34
    (1024, 2, 4, 1, 2048, True),   # 35
    (256, 4, 8, 1, 1024, True),    # 36  (c4's autotuned shape; automatic up to d = 1024)
    (192, 5, 4, 2, 0, True),       # 37  (c5's)
    # large states (d <= 3072: the gather and e buffers still fit in shared
    # memory): two history rows in registers, the rest in the per-CTA
    # overflow scratch (L2), G as CSR through L1/L2
    (1024, 3, 2, 1, 3072),         # 38
    # Nordsieck rows 2..7 and e / e_prev in TMEM (HistT, csrc/qtm_tmem.cuh):
    # 128 registers and ~110 KB of shared memory per d <= 1024 trajectory,
    # so two trajectory CTAs share an SM (each allocating 256 TMEM columns)
    (256, 4, 8, 2, 1024, False, True),   # 39  automatic for 512 < d <= 1024 (c4 1.29x over #22)
    # (its time-dependent twin needs 208 KB of shared memory for c4td's
    # union-pattern tables, so one CTA per SM: 13.2k vs #36's 15.4k; not built)
]
# one thread per trajectory for tiny states (csrc/qtm_small.cuh):
# (d_max, trajectories per warp, auto-select for dim <= this (0 = never))
# c1 (500 trajectories, ~220 strictly sequential attempts each) measured per
# step: (32,1,13) 1.09 ms; (2, 1 lane) 0.75 ms; (2, 4 lanes) 1.13 ms;
# (2, 32 lanes) 1.93 ms (divergence); (4, 1) 1.52 ms
SMALL_VARIANTS = [
    (2, 1, 2),     # 40  automatic for d <= 2 (c1)
    (2, 4, 0),     # 41  (more trajectories per warp: large ensembles)
    (4, 1, 4),     # 42  automatic for 2 < d <= 4
]

# variants added after the small ones (so the ids above stay what tests, docs
# and profiles call them): same tuple format as VARIANTS
LATE_VARIANTS = [
    # the TMEM variant with the time-dependent terms compiled in: fits two CTAs
    # per SM when the staged term needs no per-slot tables (sell_spmv_tdd:
    # c4td's modulated field is one value), else one
    (256, 4, 8, 2, 0, True, True),       # 43
]

SOURCES = ["qtm_traj.cuh", "qtm_bdf.cuh", "qtm_rng.cuh", "qtm_tmem.cuh", "qtm_small.cuh", "qtm_capi.cu"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _write_if_changed(path: str, text: str) -> None:
    if os.path.exists(path) and open(path).read() == text:
        return
    with open(path, "w") as f:
        f.write(text)


def generate() -> list[str]:
    os.makedirs(GEN, exist_ok=True)
    files = []
    decls = []
    rows = []
    def emit(i, row):
            nt, e, rr, mb, auto = row[:5]
            td = "true" if len(row) > 5 and row[5] else "false"
            tmem = "true" if len(row) > 6 and row[6] else "false"
            name = f"variant_{i}.cu"
            body = f"""// generated by build.py -- kernel variant {i}
#include "../qtm_traj.cuh"
namespace qtm {{
template __global__ void traj_kernel<{nt}, {e}, {rr}, {mb}, {td}, {tmem}>(const __grid_constant__ DevProblem,
                                                                     const __grid_constant__ RunParams);
VariantDesc variant_{i}() {{
    return VariantDesc{{{nt}, {e}, {rr}, {mb}, {auto}, {1 if td == "true" else 0},
                           TrajKernel<{nt}, {e}, {rr}, {tmem}>::smem_bytes(),
                           reinterpret_cast<const void*>(traj_kernel<{nt}, {e}, {rr}, {mb}, {td}, {tmem}>),
                           {1 if tmem == "true" else 0}, 0, 0}};
}}
}}  // namespace qtm
"""
            _write_if_changed(os.path.join(GEN, name), body)
            files.append(os.path.join(GEN, name))
            decls.append(f"VariantDesc variant_{i}();")
            rows.append(f"        variant_{i}(),")
    for i, row in enumerate(VARIANTS):
        emit(i, row)
    for j, (dmax, lanes, auto) in enumerate(SMALL_VARIANTS):
        i = len(VARIANTS) + j
        name = f"variant_{i}.cu"
        body = f"""// generated by build.py -- kernel variant {i} (one thread per trajectory)
#include "../qtm_small.cuh"
namespace qtm {{
template __global__ void traj1_kernel<{dmax}>(const __grid_constant__ DevProblem,
                                            const __grid_constant__ RunParams);
VariantDesc variant_{i}() {{
    return VariantDesc{{128, {dmax}, 13, 1, {auto}, 0, 0,
                       reinterpret_cast<const void*>(traj1_kernel<{dmax}>), 0, {dmax}, {lanes}}};
}}
}}  // namespace qtm
"""
        _write_if_changed(os.path.join(GEN, name), body)
        files.append(os.path.join(GEN, name))
        decls.append(f"VariantDesc variant_{i}();")
        rows.append(f"        variant_{i}(),")
    for j, row in enumerate(LATE_VARIANTS):
        emit(len(VARIANTS) + len(SMALL_VARIANTS) + j, row)
    table = ("// generated by build.py\nnamespace qtm {\n" + "\n".join(decls) + "\n}  // namespace qtm\n"
             "static const std::vector<qtm::VariantDesc>& qtm_variant_table() {\n"
             "    using namespace qtm;\n    static const std::vector<VariantDesc> t = {\n"
             + "\n".join(rows) + "\n    };\n    return t;\n}\n")
    _write_if_changed(os.path.join(GEN, "variant_table.inc"), table)
    return files


def _stamp(paths) -> str:
    h = hashlib.sha1()
    for p in sorted(paths):
        h.update(open(p, "rb").read())
    h.update(" ".join(NVCC_FLAGS).encode())
    h.update(repr(VARIANTS).encode())
    h.update(repr(SMALL_VARIANTS).encode())
    h.update(repr(LATE_VARIANTS).encode())
    return h.hexdigest()


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    units = generate() + [os.path.join(CSRC, "qtm_capi.cu")]
    deps = units + [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(INCLUDE, "qtm.h")]
    stamp = _stamp(deps)
    stamp_file = os.path.join(OBJ, "stamp")
    if not force and os.path.exists(LIB) and os.path.exists(stamp_file) \
            and open(stamp_file).read() == stamp:
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    exe = nvcc()

    def compile_one(src):
        obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
        cmd = [exe, *NVCC_FLAGS, "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    jobs = jobs or max(1, min(len(units), os.cpu_count() or 1))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(compile_one, units))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    tmp = LIB + ".tmp"
    r = subprocess.run([exe, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(stamp_file, "w") as f:
        f.write(stamp)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args(argv)
    print(build(force=a.force, jobs=a.jobs, verbose=a.verbose))


if __name__ == "__main__":
    main()
