"""Build-time guard (no GPU): device code must never read the host-only constexpr architecture
tables at run time.  A runtime index into a `static constexpr` LayerArch in device code compiles to
a generic load from a small constant address (the fused layer-1 kernel faulted that way, DESIGN.md
§5); every loop over irreps in device code is a compile-time static_for.  This test compiles each
translation unit to PTX and looks for generic loads whose address register holds an immediate."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2303_08169_b200", "csrc")


def _nvcc():
    return shutil.which("nvcc") or ("/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else None)


@pytest.mark.parametrize("tu", ["tp_fused.cu", "model.cu", "tc_gemm.cu", "neighbor.cu", "md.cu", "pimd.cu"])
def test_no_constant_address_generic_loads(tu, tmp_path):
    nvcc = _nvcc()
    if nvcc is None:
        pytest.skip("nvcc not available")
    out = tmp_path / (tu + ".ptx")
    r = subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
                        "-I", os.path.join(ROOT, "include"), "-ptx", os.path.join(CSRC, tu), "-o", str(out)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    imm = {}
    bad = []
    for ln in out.read_text().splitlines():
        m = re.match(r"\s*mov\.(?:u64|b64)\s+(%rd\d+),\s*(\d+);", ln)
        if m:
            imm[m.group(1)] = int(m.group(2))
            continue
        m = re.match(r"\s*ld(\.v\d)?\.(?:u|s|f|b)\d+\s+\S+,\s*\[(%rd\d+)", ln)
        if m and m.group(2) in imm and imm[m.group(2)] < 1 << 16:
            bad.append(ln.strip())
    assert not bad, bad[:5]
