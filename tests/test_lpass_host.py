"""Host logic of the relabelling tile pass (paper_1805_04708_b200/csrc/lpass.h).

The pass compiler (lpass_compile.cpp) turns a run of gates into a program of
register stages; tools/lpass_emu.cpp interprets that program on the CPU with
the kernel's semantics and compares, on random runs of every gate kind (dense,
phase, permutation, 1-2 controls in or outside the tile, global controls,
R = 4 and 5, K = 9..12), with applying the gates one by one (Eq. NUM2 with
controls).  Test infrastructure only: no GPU, no oracle.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def emu(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("lpass") / "lpass_emu")
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-o", exe,
                           os.path.join(ROOT, "tools", "lpass_emu.cpp"),
                           os.path.join(ROOT, "paper_1805_04708_b200", "csrc", "lpass_compile.cpp")])
    return exe


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_compiled_program_equals_sequential_application(emu, seed):
    out = subprocess.run([emu, "300", str(seed)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok"), out.stdout


@pytest.mark.parametrize("seed", [1, 2])
def test_scheduler_whole_circuits(emu, seed):
    """lpass_run (the runtime's pass scheduler, with diagonals carried across
    stages and deferred across passes) on whole random and layered circuits:
    terminates and equals sequential application."""
    out = subprocess.run([emu, "30", str(seed), "run"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok"), out.stdout
