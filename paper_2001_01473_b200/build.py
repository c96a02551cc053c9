"""Build libAN5D.so (sm_100a) in-tree.

Generates one translation unit per kernel instance under csrc/gen/, compiles them in parallel with
nvcc (-gencode arch=compute_100a,code=sm_100a -lineinfo), and links the shared library next to this
file.  Incremental: an object is rebuilt only when its source, a header it depends on or the flags
changed (digests use repo-relative paths, so a fresh clone anywhere rebuilds the same way).

Build-time budget (round-2 rule): a clean default build must finish in a few minutes on an 8-core
CPU box.  Hence
  * the default instance set is CORE (below): what the planner picks at BASELINE sizes plus the
    reduced degrees under each pick (~80 instances); the full b_T-sweep matrix of BASELINE configs
    2-3 (~240 instances, ~15 min) is opt-in with AN5D_FULL_BUILD=1;
  * the register budget of every known instance comes from the committed table regcaps.json, so
    nothing compiles twice; only instances missing from the table run the spill-retry loop.
"""
from __future__ import annotations

import hashlib
import json
import re
import os
import shutil
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# AN5D_BUILD_TAG builds an experimental library (own object dir, libAN5D_<tag>.so, selected at run
# time with AN5D_LIB) with AN5D_EXTRA_NVCC flags; the product library is always the untagged one.
_TAG = os.environ.get("AN5D_BUILD_TAG", "")
GEN = os.path.join(CSRC, "gen" + (f"_{_TAG}" if _TAG else ""))
OBJ = os.path.join(HERE, "build" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(HERE, f"libAN5D_{_TAG}.so" if _TAG else "libAN5D.so")
REPO = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v", "-diag-suppress", "177,836",
    "-I", "include",
] + os.environ.get("AN5D_EXTRA_NVCC", "").split()   # nvcc runs with cwd = REPO (relative paths)


# Default ("core") instance set: for every Table-2 stencil family and dtype, the (b_T, vec) the
# measured planner picked at BASELINE sizes in round 1 (profiles/r01_v9_suite.jsonl), one b_T of
# headroom where the pick sat at the HBM/FMA crossover, and every lower degree with the same vec
# (the reduced-degree sweeps of the final-block adjustment, and small-T runs).
# Key: (ndim, dtype, shape, rad) -> [(vec, max b_T)]; dtype 0 = f32, 1 = f64; shape 0 = star, 1 = box.
CORE = {
    (2, 0, 0, 1): [(8, 8)], (2, 0, 0, 2): [(8, 5)], (2, 0, 0, 3): [(8, 3)], (2, 0, 0, 4): [(8, 2)],
    (2, 0, 1, 1): [(8, 5)], (2, 0, 1, 2): [(8, 2)], (2, 0, 1, 3): [(4, 1)], (2, 0, 1, 4): [(4, 1)],
    (2, 1, 0, 1): [(4, 7)], (2, 1, 0, 2): [(4, 4)], (2, 1, 0, 3): [(4, 2)], (2, 1, 0, 4): [(4, 2)],
    (2, 1, 1, 1): [(4, 4)], (2, 1, 1, 2): [(4, 2)], (2, 1, 1, 3): [(4, 1)], (2, 1, 1, 4): [(4, 1)],
    (3, 0, 0, 1): [(2, 4)], (3, 0, 0, 2): [(2, 2)], (3, 0, 0, 3): [(2, 1)], (3, 0, 0, 4): [(2, 1)],
    (3, 0, 1, 1): [(2, 2)], (3, 0, 1, 2): [(2, 1)], (3, 0, 1, 3): [(2, 1)], (3, 0, 1, 4): [(2, 1)],
    (3, 1, 0, 1): [(2, 3)], (3, 1, 0, 2): [(2, 2)], (3, 1, 0, 3): [(2, 1)], (3, 1, 0, 4): [(2, 1)],
    (3, 1, 1, 1): [(2, 2)], (3, 1, 1, 2): [(2, 1)], (3, 1, 1, 3): [(2, 1)], (3, 1, 1, 4): [(2, 1)],
}
# partial sums OFF (direct gather, BASELINE config 4 = box2d2r fp32): vec 8 and 4, b_T 1..2
CORE_DIRECT = {(2, 0, 1, 2): [(8, 2), (4, 2)]}
# multi-field systems (NEXT N4): 2 fields advanced together, layout "x2" (NF = 2)
CORE_SYSTEM = {(2, 0, 0, 1): [(8, 4), (4, 5)], (2, 0, 1, 1): [(8, 3)], (2, 1, 0, 1): [(4, 3)], (2, 1, 1, 1): [(4, 2)]}
# gradient2d (shape 2, Table 2, NEXT N3): non-linear, direct gather only
CORE_GRAD = {(2, 0, 2, 1): [(8, 4), (4, 4)], (2, 1, 2, 1): [(4, 3)]}
# 3D 512-thread layouts (kernel3d.cuh Kernel3DTraits): "t32x2" = 32 x 16 threads with 2-cell patch
# rows (fp64: 64-wide tiles at half the registers per thread, twice the warps per SM; rad <= 2),
# "t32x4" = 32 x 16 threads with 4-cell rows (fp32: 128-wide tiles, less x-halo redundancy).
# Key as CORE -> [(vec, max b_T, layout)].
# "c2" / "c4" = the 256-thread layout in thread-block clusters of 2 / 4 blocks stacked along y
# that share their y halos through DSMEM (NEXT N2; one tile of 64 x 64 / 64 x 128 cells),
# "c2t32x2" the fp64 512-thread layout in pairs.  rad <= VY (row-band exchange).
CORE_LAYOUTS = {
    (3, 1, 0, 1): [(2, 3, "t32x2"), (2, 3, "c2"), (2, 3, "c2t32x2")],
    (3, 1, 0, 2): [(2, 2, "t32x2"), (2, 2, "c2t32x2")],
    (3, 1, 1, 1): [(2, 2, "t32x2"), (2, 2, "c2t32x2")],
    (3, 0, 0, 1): [(2, 4, "c2"), (2, 4, "c4")], (3, 0, 0, 2): [(2, 2, "c2")], (3, 0, 1, 1): [(2, 2, "c2")],
}
# "os" = output-stationary b_T = 1 tiles (kernel3d.cuh OS): threads cover only the compute region,
# neighbours are read from the staged plane (no halo cell computed, no shuffle) -- for the
# stencils whose planner pick is b_T = 1 (high radius, high-order box, fp64 box rad 1)
for _k in [(3, d, sh, r) for d in (0, 1) for sh in (0, 1) for r in (1, 2, 3, 4)
           if sh == 1 or r >= 2]:
    CORE_LAYOUTS.setdefault(_k, []).append((2, 1, "os"))
# "oy" = y-staged tiles for b_T >= 2 (kernel3d.cuh OS bit 0): the y halo the threads compute
# shrinks from b_T rad to (b_T - 1) rad; the stencils whose pick is b_T >= 2 (fp64: the 512-thread
# layout "oyt32x2")
for _k, _lst in {(3, 0, 0, 1): [(2, 4, "oy")], (3, 0, 0, 2): [(2, 2, "oy")], (3, 0, 1, 1): [(2, 2, "oy")],
                 (3, 1, 0, 1): [(2, 3, "oyt32x2"), (2, 3, "osxyt32x2")],
                 (3, 1, 0, 2): [(2, 2, "oyt32x2"), (2, 2, "osxyt32x2")],
                 (3, 1, 1, 1): [(2, 2, "oyt32x2"), (2, 2, "osxyt32x2")]}.items():
    CORE_LAYOUTS.setdefault(_k, []).extend(_lst)
# fp32 128-wide tiles: measured 5-15 % slower than two 64-wide blocks per SM (r02b suite), never
# picked by the tuner -> full build only
FULL_LAYOUTS = {
    (3, 0, 0, 1): [(2, 4, "t32x4")], (3, 0, 0, 2): [(2, 2, "t32x4")], (3, 0, 0, 3): [(2, 1, "t32x4")],
    (3, 0, 0, 4): [(2, 1, "t32x4")], (3, 0, 1, 1): [(2, 2, "t32x4")],
}
# 3D layout -> (TXT, VX, CL[, OS]): threads along x, cells per thread along x, blocks per cluster
# along y, output-stationary b_T = 1 tiles
LAYOUTS = {"": (16, 4, 1), "t32x2": (32, 2, 1), "t32x4": (32, 4, 1), "c2": (16, 4, 2), "c4": (16, 4, 4),
           "c2t32x2": (32, 2, 2), "os": (16, 4, 1, 3), "oy": (16, 4, 1, 1), "oyt32x2": (32, 2, 1, 1),
           "osxyt32x2": (32, 2, 1, 3)}
# 2D level split "w2" (kernel2d.cuh Split2D): two warps per tile, warp 0 levels 1..b_T/2 with the
# staging, warp 1 the rest with the store -- half the partial-sum registers per warp.  b_T 1 has
# nothing to split: the reduced-degree sweep of degree 1 uses the one-warp instance.
# Measured on B200 (profiles/r02d_split2d.jsonl): 8-13 % SLOWER than one warp per tile for
# every stencil tried, so the default build keeps only star2d1r (tests, bench --nthr 64) and the
# full build the rest.
CORE_SPLIT = {(2, 0, 0, 1): [(8, 8)]}
FULL_SPLIT = {(2, 0, 0, 2): [(8, 6)], (2, 0, 1, 1): [(8, 6)], (2, 1, 0, 1): [(4, 7)], (2, 1, 0, 2): [(4, 5)]}


def full_instances():
    """The full matrix (BASELINE configs 2-3 b_T sweeps: 2D b_T 1..10, 3D b_T 1..6), AN5D_FULL_BUILD=1.
    Register-tiling factors and b_T ranges are limited to configurations whose register queue fits
    the 255-register budget:
      2D: fp32 vec 8 (rad*bT <= 10) and vec 4 (rad*bT <= 12); fp64 vec 4 (rad*bT <= 10) and
          vec 2 (rad <= 2, rad*bT <= 4).
      3D: fp32 vy 4 (rad*bT <= 4, not box rad >= 2), vy 2 (rad*bT <= 8); fp64 vy 2 (rad*bT <= 4).
      2D box direct-gather variant: fp32 vec 8 and vec 4, fp64 vec 4, rad*bT <= 8."""
    out = []
    for shape in (0, 1):
        for rad in range(1, 5):
            for bT in range(1, 11):
                if rad * bT <= 10:
                    out.append((2, 0, shape, rad, bT, 8))
                if rad * bT <= 12:
                    out.append((2, 0, shape, rad, bT, 4))
                if rad * bT <= 10:
                    out.append((2, 1, shape, rad, bT, 4))
                if rad <= 2 and rad * bT <= 4:
                    out.append((2, 1, shape, rad, bT, 2))
                if shape == 1 and rad * bT <= 8:
                    out += [(2, 0, 1, rad, bT, 8, 0), (2, 0, 1, rad, bT, 4, 0), (2, 1, 1, rad, bT, 4, 0)]
            for bT in range(1, 7):
                if rad * bT <= 4 and not (shape == 1 and rad >= 2):
                    out.append((3, 0, shape, rad, bT, 4))
                if rad * bT <= 8:
                    out.append((3, 0, shape, rad, bT, 2))
                if rad * bT <= 4:
                    out.append((3, 1, shape, rad, bT, 2))
    return [(i + ("",)) if len(i) == 7 else i + (1, "") for i in out]


def core_instances():
    out = []
    for tab, assoc in ((CORE, 1), (CORE_DIRECT, 0), (CORE_GRAD, 0)):
        for (ndim, dtype, shape, rad), lst in tab.items():
            for vec, bmax in lst:
                out += [(ndim, dtype, shape, rad, bT, vec, assoc, "") for bT in range(1, bmax + 1)]
    for (ndim, dtype, shape, rad), lst in CORE_LAYOUTS.items():
        for vec, bmax, lay in lst:
            out += [(ndim, dtype, shape, rad, bT, vec, 1, lay) for bT in range(1, bmax + 1)]
    for (ndim, dtype, shape, rad), lst in CORE_SYSTEM.items():
        for vec, bmax in lst:
            out += [(ndim, dtype, shape, rad, bT, vec, 1, "x2") for bT in range(1, bmax + 1)]
    for (ndim, dtype, shape, rad), lst in CORE_SPLIT.items():
        for vec, bmax in lst:
            out += [(ndim, dtype, shape, rad, bT, vec, 1, "w2") for bT in range(2, bmax + 1)]
    return out


def instances():
    """(ndim, dtype, shape, rad, bT, vec, assoc, layout) tuples; dtype 0=f32 1=f64, shape 0=star
    1=box, assoc 1 = partial sums, 0 = direct gather, layout "" or a 3D LAYOUTS key.  Default: core_instances(); AN5D_FULL_BUILD=1: the
    full b_T-sweep matrix (plus the core set); AN5D_DEV_INSTANCES: a development subset."""
    out = core_instances()
    if os.environ.get("AN5D_FULL_BUILD", "") not in ("", "0"):
        extra = [(nd, dt, sh, r, bT, v, 1, "w2") for (nd, dt, sh, r), lst in FULL_SPLIT.items()
                 for v, bmax in lst for bT in range(2, bmax + 1)]
        extra += [(nd, dt, sh, r, bT, v, 1, lay) for (nd, dt, sh, r), lst in FULL_LAYOUTS.items()
                  for v, bmax, lay in lst for bT in range(1, bmax + 1)]
        out = sorted(set(out) | set(full_instances()) | set(extra))
    dev = os.environ.get("AN5D_DEV_INSTANCES")
    if dev:
        # quick development subset: comma list of "ndim:dtype:shape:rad" groups, or "min"
        if dev == "min":
            keep = {(2, 0, 0, 1), (2, 1, 0, 1), (2, 0, 1, 1), (3, 0, 0, 1), (3, 0, 1, 1)}
        else:
            keep = {tuple(int(v) for v in g.split(":")) for g in dev.split(",")}
        out = [i for i in out if i[:4] in keep]
    return out


def inst_name(ndim, dtype, shape, rad, bT, vec, assoc, layout=""):
    return (f"inst_{ndim}d_{'f64' if dtype else 'f32'}_{('star', 'box', 'grad')[shape]}_r{rad}"
            f"_bt{bT}_v{vec}{'' if assoc else '_direct'}{'_' + layout if layout else ''}")


def _regcaps():
    with open(os.path.join(HERE, "regcaps.json")) as f:
        return json.load(f)["caps"]


def generate():
    """One generated translation unit per kernel instance (balanced parallel compilation).  The
    instance's calibrated register cap (regcaps.json) is baked into its source."""
    os.makedirs(GEN, exist_ok=True)
    caps = _regcaps()
    files = []
    for inst in instances():
        (ndim, dtype, shape, rad, bT, vec, assoc, layout) = inst
        T = "double" if dtype else "float"
        name = inst_name(*inst)
        targs = f"{T}, {rad}, {bT}, {vec}, {'true' if shape == 1 else 'false'}" + ("" if assoc else ", false")
        if shape == 2:
            targs += ", 1, true"   # gradient2d (GRAD template flag)
        if layout == "w2":
            targs += ", true, 2"
        elif layout == "x2":
            targs += ", true, 1, false, 2"   # NF = 2 fields
        elif layout:
            lay = LAYOUTS[layout]
            targs += ", %d, %d, %d" % lay[:3] + (", %d" % lay[3] if len(lay) > 3 and lay[3] else "")
        fn = "make_instance2d" if ndim == 2 else "make_instance3d"
        lines = ["// GENERATED by paper_2001_01473_b200/build.py -- one kernel instance."]
        if name in caps:
            lines.append("// register cap calibrated in regcaps.json (compiled once, no spill retry)")
            lines.append("#define AN5D_CAP_KNOWN 1")
            if caps[name] is not None:
                lines.append(f"#define AN5D_MINB_CAP {int(caps[name])}")
        lines += [
            f'#include "../inst{ndim}d.cuh"',
            "namespace an5d {",
            "namespace {",
            f"Registrar reg({fn}<{targs}>());",
            "}  // namespace",
            "}  // namespace an5d",
            "",
        ]
        text = "\n".join(lines)
        path = os.path.join(GEN, name + ".cu")
        if not os.path.exists(path) or open(path).read() != text:
            with open(path, "w") as f:
                f.write(text)
        files.append(path)
    # drop stale generated files
    for f in os.listdir(GEN):
        p = os.path.join(GEN, f)
        if p not in files:
            os.remove(p)
    return files


# headers each kind of translation unit depends on (a 2D change does not rebuild the 3D instances)
DEPS = {
    "2d": ["args.hpp", "common.cuh", "lane.cuh", "registry.hpp", "kernel2d.cuh", "inst2d.cuh"],
    "3d": ["args.hpp", "common.cuh", "lane.cuh", "registry.hpp", "kernel3d.cuh", "inst3d.cuh"],
    "host": None,   # every header
}


def _header_digest(kind="host"):
    h = hashlib.sha1()
    names = DEPS[kind] or sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h")))
    for f in names:
        h.update(open(os.path.join(CSRC, f), "rb").read())
    if kind == "host":   # the kernel instances do not include the C ABI header
        h.update(open(os.path.join(REPO, "include", "an5d.h"), "rb").read())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


SPILL_LIMIT = 32   # bytes of spill stores tolerated before the register cap is relaxed


def _spill_bytes(log):
    return max([int(v) for v in re.findall(r"(\d+) bytes spill stores", log)] or [0])


def _compile(src, nvcc, hdr):
    """Compile one translation unit.  Instances with a calibrated cap (regcaps.json) compile once.
    Unlisted instances: if ptxas reports more than SPILL_LIMIT bytes of spill stores, retry with a
    lower minimum-blocks cap (a larger register budget) and report the cap to add to the table."""
    base = os.path.splitext(os.path.basename(src))[0]
    obj = os.path.join(OBJ, base + ".o")
    stamp = obj + ".sha"
    text = open(src, "rb").read()
    digest = hashlib.sha1(text + hdr.encode()).hexdigest()
    if os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == digest:
        return obj, None
    known = b"AN5D_CAP_KNOWN" in text or "inst_" not in base
    rel = os.path.relpath(src, REPO)
    logs = []
    cap = None
    t0 = time.time()
    while True:
        extra = [] if cap is None else [f"-DAN5D_MINB_CAP={cap}"]
        cmd = [nvcc] + NVCC_FLAGS + extra + ["-c", rel, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True, cwd=REPO)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
        logs.append(f"# AN5D_MINB_CAP={cap}\n" + r.stderr)
        regs = max([int(v) for v in re.findall(r"Used (\d+) registers", r.stderr)] or [255])
        if known or "AN5D_MINB_FORCE" in " ".join(NVCC_FLAGS) or _spill_bytes(r.stderr) <= SPILL_LIMIT or regs > 168:
            break
        # next register budget (minimum resident blocks): 2D one-warp blocks 16 -> 12 -> 1
        # (128 -> 168 -> 255 registers), two-warp blocks 8 -> 6 -> 3, 3D 2 -> 1.  A 512-thread 3D
        # layout is already at one block (<= 128 registers): nothing left to relax
        if "_w2" in base:
            ladder = [6, 3]
        elif "_2d_" in base:
            ladder = [12, 1]
        else:
            ladder = [1]
        nxt = next((c for c in ladder if regs < {12: 168, 1: 255, 6: 168, 3: 255}[c]), None)
        if nxt is None or nxt == cap or "_t32x" in base:
            break
        cap = nxt
    if not known:
        print(f"build.py: {base} not in regcaps.json; calibrated cap = {cap} (add it to the table)",
              file=sys.stderr)
    with open(obj + ".ptxas.log", "w") as f:
        f.write(f"# wall {time.time() - t0:.1f} s\n" + "\n".join(logs))
    with open(stamp, "w") as f:
        f.write(digest)
    return obj, logs[-1]


def build(jobs: int | None = None, verbose: bool = True) -> str:
    t0 = time.time()
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    os.makedirs(OBJ, exist_ok=True)
    srcs = generate() + [os.path.join(CSRC, "an5d_host.cu"), os.path.join(CSRC, "an5d_model.cu")]
    hdr = {k: _header_digest(k) for k in DEPS}
    jobs = jobs or max(1, os.cpu_count() or 1)
    # heavy instances (3D, box, high b_T) first so the longest compiles do not end up in the tail
    def weight(s):
        m = re.search(r"_r(\d)_bt(\d+)_", s)
        return (("_3d_" in s) * 4 + ("_box_" in s) * 2 + (int(m.group(1)) * int(m.group(2)) if m else 99))
    srcs.sort(key=weight, reverse=True)
    kind = lambda s: "2d" if "inst_2d_" in s else ("3d" if "inst_3d_" in s else "host")
    with ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, nvcc, hdr[kind(s)])[0], srcs))
    stamp = os.path.join(OBJ, "lib.sha")
    digest = hashlib.sha1("".join(sorted(open(o + ".sha").read() for o in objs)).encode()).hexdigest()
    if os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == digest:
        return LIB
    tmp = LIB + ".tmp"
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs + ["-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(digest)
    if verbose:
        print(f"built {LIB} ({len(srcs) - 2} kernel instances, {jobs} jobs, {time.time() - t0:.0f} s)",
              file=sys.stderr)
    return LIB


def update_caps():
    """Record the cap each built instance ended with (its ptxas log) in regcaps.json."""
    path = os.path.join(HERE, "regcaps.json")
    with open(path) as f:
        d = json.load(f)
    for inst in instances():
        name = inst_name(*inst)
        log = os.path.join(OBJ, name + ".o.ptxas.log")
        if name in d["caps"] or not os.path.exists(log):
            continue
        caps = re.findall(r"# AN5D_MINB_CAP=(\S+)", open(log).read())
        d["caps"][name] = None if not caps or caps[-1] == "None" else int(caps[-1])
    d["caps"] = dict(sorted(d["caps"].items()))
    with open(path, "w") as f:
        json.dump(d, f, indent=1)


if __name__ == "__main__":
    if "--update-caps" in sys.argv:
        update_caps()
    else:
        build()
