"""Codegen guard for the headline executor (CPU: nvcc cross-compiles).

The streamed push-form kernel runs at the 72-register cap that gives 7 CTAs
per SM; a few bytes of register spills in its block loop cost ~15 % at C5
(measured: 1.29 -> 1.53 ms when an unrelated field grew the kernel's
parameter struct).  This reads the ``-Xptxas -v`` report the build keeps for
exec_hier_stream.cu (compiling it when missing or stale) and requires the C5 / C1 headline instantiation
(``hier_stream_kernel<OpFlux, double, AoS, colour, u8 slots, 2 rows/thread,
LDGSTS, staged reads, push>``) to spill nothing.
"""

import re
import shutil
import subprocess

import pytest

from conftest import REPO

HEADLINE = "hier_stream_kernelINS_6OpFluxEdLi0ELb0EhLi2ELb0ELb1ELb0ELb0EEEv"


@pytest.mark.skipif(shutil.which("nvcc") is None and not (REPO / "build").exists(), reason="no nvcc")
def test_headline_executor_does_not_spill(tmp_path):
    from paper_1802_03749_b200 import build_native as bn

    src = bn.CSRC / "exec_hier_stream.cu"
    log = bn.OBJ_DIR / (src.name + ".ptxas.txt")  # written by every build (build_native._compile)
    if log.exists() and log.stat().st_mtime >= max(src.stat().st_mtime, bn._headers_mtime()):
        text = log.read_text()
    else:
        cmd = [bn._nvcc(), *bn.NVCC_FLAGS, "-Xptxas", "-v", "-c", str(src), "-o", str(tmp_path / "s.o")]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        text = r.stderr
    lines = text.splitlines()
    idx = [i for i, l in enumerate(lines) if "Compiling entry function" in l and HEADLINE in l]
    assert idx, "headline instantiation not found"
    block = " ".join(lines[idx[0]:idx[0] + 4])
    spill = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", block)
    regs = re.search(r"Used (\d+) registers", block)
    assert spill and spill.groups() == ("0", "0"), block
    assert regs and int(regs.group(1)) <= 72, block
