"""The App. B instruction language: the host parser
(qsim_asm_parse, no GPU).  Gate matrices are compared with the generator's
App. B matrices (qsim_inputs, pinned in test_circuits.py)."""
import math

import numpy as np
import pytest

import paper_1805_04708_b200 as q
import qsim_inputs as C


def _one(text):
    d = q.asm_parse("QUBITS 4\n" + text)
    assert len(d["ops"]) == 1
    return d["ops"][0]


@pytest.mark.parametrize("mn,mat", [("H", C.mat_H()), ("X", C.mat_X()), ("Y", C.mat_Y()), ("Z", C.mat_Z()),
                                    ("S", C.mat_S()), ("S+", C.mat_S(True)), ("T", C.mat_T()),
                                    ("T+", C.mat_T(True)), ("+X", C.mat_pX(+1)), ("-X", C.mat_pX(-1)),
                                    ("+Y", C.mat_pY(+1)), ("-Y", C.mat_pY(-1))])
def test_single_qubit_mnemonics(mn, mat):
    o = _one(f"{mn} 2")
    assert o["type"] == q.ASM_GATE and o["target"] == 2 and o["controls"] == []
    assert np.max(np.abs(o["u"] - mat)) <= 1e-15


def test_parametrised_gates_and_phases():
    assert np.max(np.abs(_one("U1 1 0.7")["u"] - C.mat_U1(0.7))) <= 1e-15
    assert np.max(np.abs(_one("U2 1 0.3 -1.1")["u"] - C.mat_U2(0.3, -1.1))) <= 1e-15
    assert np.max(np.abs(_one("U3 1 2.0 0.3 -1.1")["u"] - C.mat_U3(2.0, 0.3, -1.1))) <= 1e-15
    for k in (0, 1, 3, -2, -5):
        assert np.max(np.abs(_one(f"R 3 {k}")["u"] - C.mat_R(k))) <= 1e-15
    o = _one("U 0 3 -4")  # U(k) with k < 0 is U^dagger
    assert o["target"] == 3 and o["controls"] == [0]
    assert np.max(np.abs(o["u"] - C.mat_R(-4))) <= 1e-15
    o = _one("CNOT 2 1")
    assert o["target"] == 1 and o["controls"] == [2] and np.array_equal(o["u"], C.mat_X())
    o = _one("TOFFOLI 0 3 1")
    assert o["target"] == 1 and o["controls"] == [0, 3] and np.array_equal(o["u"], C.mat_X())


def test_control_instructions_comments_and_case():
    d = q.asm_parse("""! a comment line
qubits 6      ! trailing comment
BIT ASSIGNMENT 5 4 3 2 1 0
DEPOLARIZING CHANNEL P_Z = 0.25 , P_X=0.5, SEED = 9
i 0
h 1
BEGIN MEASUREMENT
M 2
SHORBOX 3 7 2
clear 4
SET 5
GENERATE EVENTS 100 -1
EXIT
""")
    assert d["n"] == 6 and d["perm"] == [5, 4, 3, 2, 1, 0]
    assert d["depol"] == [0.5, 0.0, 0.25, 9.0]
    types = [o["type"] for o in d["ops"]]  # I is a no-operation
    assert types == [q.ASM_GATE, q.ASM_MEASURE_ALL, q.ASM_M, q.ASM_SHORBOX, q.ASM_CLEAR, q.ASM_SET, q.ASM_EVENTS,
                     q.ASM_EXIT]
    assert [o["line"] for o in d["ops"]] == [6, 7, 8, 9, 10, 11, 12, 13]
    assert d["ops"][3]["args"] == [3, 7, 2] and d["ops"][6]["args"][:2] == [100, -1]


@pytest.mark.parametrize("text,line", [
    ("H 0", 1),                                   # QUBITS must come first
    ("QUBITS 1", 1), ("QUBITS 64", 1),            # 1 < N < 64
    ("QUBITS 3\nQUBITS 3", 2),
    ("QUBITS 3\nH 3", 2), ("QUBITS 3\nH -1", 2), ("QUBITS 3\nH", 2),
    ("QUBITS 3\nCNOT 1 1", 2), ("QUBITS 3\nTOFFOLI 0 0 1", 2),
    ("QUBITS 3\nU 0 1 x", 2), ("QUBITS 3\nU1 0 abc", 2),
    ("QUBITS 3\nH 0\nBIT ASSIGNMENT 0 1 2", 3), ("QUBITS 3\nBIT ASSIGNMENT 0 0 1", 2),
    ("QUBITS 3\nBIT ASSIGNMENT 0 1", 2),
    ("QUBITS 3\nDEPOLARIZING CHANNEL P_X = 0.7, P_Y = 0.5", 2),
    ("QUBITS 3\nDEPOLARIZING CHANNEL P_Q = 0.1", 2),
    ("QUBITS 3\nGENERATE EVENTS 0 1", 2), ("QUBITS 3\nSHORBOX 3 7 2", 2), ("QUBITS 3\nSHORBOX 2 7 7", 2),
    ("QUBITS 3\nFOO 1", 2), ("QUBITS 3\nEXIT 1", 2), ("", 0),
])
def test_errors_name_the_line(text, line):
    with pytest.raises(q.QsimError) as e:
        q.asm_parse(text)
    assert e.value.code == q.QSIM_EINVAL
    assert f"line {line}:" in str(e.value)
