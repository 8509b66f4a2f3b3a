"""The kernel variants DESIGN.md reports measurements for (rejected, so archived in
tools/r1_variants/ and tools/exh_tc/, not part of libpt.so) still compile for sm_100a
against the library's headers (no GPU needed: nvcc cross-compiles).  Each is built in
its own process, in parallel, as an object file."""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SRC = os.path.join(ROOT, "tools", "r1_variants", "exhaustive_variants.cu")
TC_SRC = os.path.join(ROOT, "tools", "exh_tc", "exh_tc.cu")
CSRC = os.path.join(ROOT, "paper_2507_15277_b200", "csrc")

VARIANTS = {
    "tensor_summed_mma": ["-DXT_MMA=1"],
    "tensor_summed_tiled": ["-DXT_TC=1"],
    "hybrid_sets": ["-DXT_TC=2"],
    "hybrid_relu": ["-DXT_TC=3"],
    "warp_specialised": ["-DXW_ENABLE=1"],
    "producer_warp": ["-DXT_NOPROD=0"],
    "half_rings": ["-DXT_HALF=1"],
    "wait_backoff": ["-DXT_WAITNS=256"],
    "probe": ["-DXT_PROBE=2"],
    "shape_4x8": ["-DXT_SHAPE48=1"],
    "archived_default": [],
}


@pytest.mark.skipif(not os.path.exists(NVCC) and shutil.which("nvcc") is None, reason="no nvcc")
def test_opt_in_variants_compile():
    nvcc = NVCC if os.path.exists(NVCC) else shutil.which("nvcc")
    with tempfile.TemporaryDirectory() as tmp:
        procs = {}
        for name, flags in VARIANTS.items():
            cmd = [nvcc, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                   "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "--expt-relaxed-constexpr", "-c", SRC,
                   "-o", os.path.join(tmp, name + ".o")] + flags
            procs[name] = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        procs["tcgen05_summed"] = subprocess.Popen(
            [nvcc, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
             "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "--expt-relaxed-constexpr", "-c", TC_SRC,
             "-o", os.path.join(tmp, "tc.o")], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
        failed = {}
        for name, p in procs.items():
            out, _ = p.communicate(timeout=600)
            if p.returncode != 0:
                failed[name] = out[-2000:]
        assert not failed, failed
