"""CPU-side checks of the C-ABI library: it loads, exports every symbol
include/qsim.h declares, refuses to compute without a GPU (no CPU fallback),
and its host-only planner (a2, a7) produces valid plans."""
import os
import re

import numpy as np
import pytest

import qsim_inputs as C

q = pytest.importorskip("paper_1805_04708_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "qsim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qsim_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(q.lib(), s), s
    assert set(syms) == set(q.EXPORTS)


def test_library_is_sm100a_and_in_tree():
    assert q.lib_path().startswith(ROOT)
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", q.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(q.QsimError) as e:
        q.State(10)
    assert e.value.code == q.QSIM_ECUDA


def test_gate_record_layout():
    arr, n = q.pack_gates(C.config(0, seed=1))
    assert n == 200
    c = C.config(0, seed=1)
    for i in (0, 57, 199):
        assert arr[i].target == c.target[i] and arr[i].ncontrols == c.nctrl[i]
        assert np.allclose(list(arr[i].u), c.u[8 * i:8 * i + 8])


def _apply_plan_numpy(n, P, circ, ops, final_map):
    """Execute a plan on a numpy vector in PHYSICAL order; return it in logical order."""
    nl = n - int(np.log2(P))
    v = np.zeros(1 << n, dtype=np.complex128)
    v[0] = 1
    idx = np.arange(1 << n)
    for o in ops:
        if o["type"] in (q.OP_EXCHANGE, q.OP_REMAP):  # a REMAP group = disjoint bit transpositions
            g, l = o["g"], o["l"]
            assert g >= nl and l < nl
            bg, bl = (idx >> g) & 1, (idx >> l) & 1
            j = idx & ~((1 << g) | (1 << l)) | (bg << l) | (bl << g)
            v = v[j]
        else:
            _, kind, t, t2, ctl, u = circ.gate(o["gate_index"])
            pt = o["l"]
            # only diagonal gates and relabels (permutations among global bits) stay on global bits;
            # in the physical-index view a relabel is the gate itself
            assert o["cls"] == 1 or pt < nl or o["type"] == q.OP_RELABEL
            if o["type"] == q.OP_RELABEL:
                assert pt >= nl and all(c >= nl for c in o["controls"]) and o["cls"] == 2
            cm = 0
            for c in o["controls"]:
                cm |= 1 << c
            sel = (((idx >> pt) & 1) == 0) & ((idx & cm) == cm)
            i0 = idx[sel]
            i1 = i0 | (1 << pt)
            x, y = v[i0].copy(), v[i1].copy()
            v[i0] = u[0, 0] * x + u[0, 1] * y
            v[i1] = u[1, 0] * x + u[1, 1] * y
    # physical -> logical
    L = np.zeros(1 << n, dtype=np.int64)
    for qq in range(n):
        L |= ((idx >> final_map[qq]) & 1) << qq
    out = np.empty_like(v)
    out[L] = v
    return out


@pytest.mark.parametrize("P", [2, 4, 8])
def test_planner_plan_reproduces_the_circuit(P):
    import oracle

    n = 11
    circ = C.global_permutations(n, P, seed=P)
    circ.extend(C.config(0, n=n, seed=P))
    circ.extend(C.layered(n, 1, seed=P, h_first=False))
    circ.swap(0, n - 1)
    circ.extend(C.global_permutations(n, P, seed=P + 1))
    ops, fmap = q.qsim_plan(n, P, circ)
    nex = sum(o["type"] in (q.OP_EXCHANGE, q.OP_REMAP) for o in ops)
    assert nex > 0
    assert sum(o["type"] == q.OP_RELABEL for o in ops) > 0
    if P >= 4:  # the layered part targets every global qubit: one all-to-all remap
        assert sum(o["type"] == q.OP_REMAP for o in ops) >= 2
    got = _apply_plan_numpy(n, P, circ, ops, fmap)
    assert np.max(np.abs(got - oracle.e_simulate(n, circ))) <= 1e-12


@pytest.mark.parametrize("P", [4, 8, 16])
def test_planner_remap_groups(P):
    """Config-3 recipe: every layer hits all log2(P) global qubits with dense
    gates; the planner swaps them in with one all-to-all per layer (REMAP
    groups of m = log2(P) disjoint (global, local) pairs, distinct bits, the
    gate that triggered it then local), and the plan reproduces the circuit."""
    import oracle

    n = 12
    k = int(np.log2(P))
    circ = C.layered(n, 3, seed=3)
    ops, fmap = q.qsim_plan(n, P, circ)
    nl = n - k
    groups = {}
    for o in ops:
        if o["type"] == q.OP_REMAP:
            groups.setdefault(o["gate_index"], []).append((o["g"], o["l"]))
    nx = sum(o["type"] == q.OP_EXCHANGE for o in ops)
    assert len(groups) >= 3 and len(groups) > nx
    for gi, pairs in groups.items():
        gs, ls = [p[0] for p in pairs], [p[1] for p in pairs]
        # at most 3 bits per all-to-all (the remap kernels' partner tables hold 7 partners)
        assert 2 <= len(pairs) <= min(k, 3) and len(set(gs)) == len(gs) and all(nl <= x < n for x in gs)
        assert len(set(ls)) == len(ls) and all(x < nl for x in ls)
    got = _apply_plan_numpy(n, P, circ, ops, fmap)
    assert np.max(np.abs(got - oracle.e_simulate(n, circ))) <= 1e-12


def test_planner_rejects_bad_gates():
    c = [(C.mat_H(), 7)]
    with pytest.raises(q.QsimError):
        q.qsim_plan(5, 1, c)
    with pytest.raises(q.QsimError) as e:
        q.qsim_plan(5, 1, [(np.array([[1, 1], [0, 1]]), 0)])
    assert e.value.code == q.QSIM_ENOTUNITARY
