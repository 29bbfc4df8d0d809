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


# the register-set lookahead and the pass-former search run by default only on
# large states (>= 1024 tiles); the emulator's cases are small, so they are
# also checked with both forced on
FORCED = {"LPASS_LOOKAHEAD": "1", "LPASS_SEARCH": "3"}


@pytest.mark.parametrize("forced", [False, True])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_compiled_program_equals_sequential_application(emu, seed, forced):
    env = dict(os.environ, **FORCED) if forced else None
    out = subprocess.run([emu, "300", str(seed)], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok"), out.stdout


@pytest.mark.parametrize("forced", [False, True])
@pytest.mark.parametrize("seed", [1, 2])
def test_scheduler_whole_circuits(emu, seed, forced):
    """lpass_run (the runtime's pass scheduler, with diagonals carried across
    stages and deferred across passes) on whole random and layered circuits:
    terminates and equals sequential application."""
    # LPASS_HOIST=1: the per-tile hoisting on these small states too (auto: >= 1024 tiles)
    env = dict(os.environ, LPASS_HOIST="1", **(FORCED if forced else {}))
    out = subprocess.run([emu, "30", str(seed), "run"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok"), out.stdout
    # the QFT-like ladders exercise the per-tile hoisting (phase terms on
    # full-index bits, tile scalars applied at the store)
    stats = dict(kv.split("=") for kv in out.stdout.split()[1:])
    assert int(stats["hoisted"]) > 0 and int(stats["tile_scalars"]) > 0, out.stdout


def test_specialised_kernel_sources_compile(emu, tmp_path):
    """The CUDA sources the runtime hands to NVRTC for its specialised pass
    kernels (lpass_jit_source: literal stages and ops around lpass_dev.cuh)
    compile for sm_100a with NVRTC, here on the CPU, for the first passes of
    the config-2 circuit (N = 30) -- the compile the GPU box does at run time."""
    import re
    import sys

    nvrtc = pytest.importorskip("cuda.bindings.nvrtc")
    sys.path.insert(0, ROOT)
    import qsim_inputs as C
    from paper_1805_04708_b200 import _build

    _build.gen_jit_sources()
    circ = C.config(1)
    gf = tmp_path / "cfg2.txt"
    with open(gf, "w") as f:
        for i in range(len(circ)):
            _, _, t, _, ctl, u = circ.gate(i)
            cc = list(ctl) + [-1, -1]
            z = u.reshape(-1)
            f.write("%d %d %d %d " % (t, len(ctl), cc[0], cc[1]) +
                    " ".join("%.17g %.17g" % (x.real, x.imag) for x in z) + "\n")
    out = subprocess.run([emu, "jitsrc", str(gf), "30", str(tmp_path), "2"], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.startswith("ok sources=2"), out.stdout + out.stderr
    inc = open(os.path.join(ROOT, "paper_1805_04708_b200", "csrc", "lpass_jit_src.inc")).read()

    def lit(var):
        m = re.search(r"static const char \*%s =\n(.*?)LPJ\";\n" % var, inc, re.S)
        return "".join(re.findall(r'R"LPJ\((.*?)\)LPJ"', m.group(1) + 'LPJ"', re.S))

    hdrs = [lit("kLpassTypesSrc").encode(), lit("kLpassDevSrc").encode()]
    prelude = ("typedef unsigned char uint8_t;\ntypedef unsigned short uint16_t;\ntypedef unsigned int uint32_t;\n"
               "typedef unsigned long long uint64_t;\ntypedef signed char int8_t;\ntypedef short int16_t;\n"
               "typedef int int32_t;\ntypedef long long int64_t;\n")
    for k in range(2):
        src = prelude + open(tmp_path / f"jit_{k}.cu").read()
        assert "lp_stage<4, 12, JitOps0<4>, 128, 1>" in src and "constexpr qsim::LOp" in src
        err, prog = nvrtc.nvrtcCreateProgram(src.encode(), b"lpass_jit.cu", 2, hdrs,
                                             [b"lpass_types.h", b"lpass_dev.cuh"])
        opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-default-device"]
        (err,) = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
        if err != nvrtc.nvrtcResult.NVRTC_SUCCESS:
            _, n = nvrtc.nvrtcGetProgramLogSize(prog)
            log = b" " * n
            nvrtc.nvrtcGetProgramLog(prog, log)
            pytest.fail(log.decode()[:4000])
        _, n = nvrtc.nvrtcGetCUBINSize(prog)
        assert n > 0
