"""App. B programs run on the GPU (qsim_asm_run) vs the oracle executing the
same instruction semantics: the error-correction circuit of Fig. 2 / App. C
(PAPER.md:1538-1575), BIT ASSIGNMENT invariance, the depolarising channel at
p_x = 1 (deterministic), sharded and A runs."""
import numpy as np
import pytest

import oracle
import paper_1805_04708_b200 as q
import qsim_inputs as C

pytestmark = pytest.mark.gpu

# Fig. 2: prepare qubit 0, encode into 0,1,2, flip qubit 0, measure the
# syndrome on 3,4, correct with TOFFOLIs, reset 3 to |0> and 4 to |1>.
EC = """QUBITS 5
{assign}
H 0
T 0
H 0
CNOT 0 1
CNOT 0 2
BEGIN MEASUREMENT
X 0                 ! the single-qubit error
CNOT 0 3
CNOT 1 3
CNOT 0 4
CNOT 2 4
M 3
M 4
TOFFOLI 3 4 0
X 4
TOFFOLI 3 4 1
X 3
X 4
TOFFOLI 3 4 2
X 3
H 3
H 4
CLEAR 3
SET 4
BEGIN MEASUREMENT
GENERATE EVENTS 4096 77
"""


# the instructions EC uses, read here independently of the library's parser:
# matrices from the App. B table (qsim_inputs), CNOT /
# TOFFOLI = X on the last operand controlled by the others
_GATES = {"H": C.mat_H, "T": C.mat_T, "X": C.mat_X}


def _oracle_run(text, seed):
    """The instruction semantics of App. B on the state-vector oracle."""
    lines = [ln.split("!")[0].split() for ln in text.splitlines()]
    lines = [ln for ln in lines if ln]
    assert lines[0][0] == "QUBITS" and not any(ln[0] == "BIT" for ln in lines)
    n = int(lines[0][1])
    a = oracle.e_init(n)
    tables, outcomes = [], []
    u = C.splitmix_uniform(seed, 64)
    k = 0
    for ln in lines[1:]:
        op, args = ln[0], [int(x) for x in ln[1:] if x.lstrip("-").isdigit()]
        if op in _GATES:
            a = oracle.e_apply(a, n, _GATES[op](), args[0], [])
        elif op in ("CNOT", "TOFFOLI"):
            a = oracle.e_apply(a, n, C.mat_X(), args[-1], args[:-1])
        elif op == "BEGIN":
            tables.append(oracle.e_expectations(a, n))
        elif op == "M":
            out, _ = oracle.e_measure(a, n, args[0], u[k])
            outcomes.append((args[0], out))
            k += 1
        elif op in ("CLEAR", "SET"):
            assert oracle.e_project(a, n, args[0], 1 if op == "SET" else 0) == 0
        elif op == "GENERATE":
            break
        else:
            raise AssertionError(f"instruction not modelled here: {op}")
    return np.array(tables), outcomes, a


@pytest.mark.parametrize("seed", [0, 5])
def test_error_correction_program(seed):
    text = EC.format(assign="")
    got = q.asm_run(text, seed=seed)
    tab, outs, a = _oracle_run(text, seed)
    assert got["outcomes"] == outs
    assert np.max(np.abs(got["tables"] - tab.reshape(got["tables"].shape))) <= 1e-12
    # the error is corrected: qubits 0..2 end as they were encoded; CLEAR / SET
    assert np.max(np.abs(got["tables"][1, :3] - got["tables"][0, :3])) <= 1e-12
    assert abs(got["tables"][1, 3, 2] - 0.0) <= 1e-12 and abs(got["tables"][1, 4, 2] - 1.0) <= 1e-12
    ev = got["events"]
    assert len(ev) == 4096
    p = np.abs(a) ** 2
    assert np.all(p[ev.astype(np.int64)] > 1e-12)  # every event is a possible basis state


def test_bit_assignment_leaves_results_unchanged():
    a = q.asm_run(EC.format(assign=""), seed=3)
    b = q.asm_run(EC.format(assign="BIT ASSIGNMENT 4 2 0 3 1"), seed=3)
    assert a["outcomes"] == b["outcomes"]
    assert np.max(np.abs(a["tables"] - b["tables"])) <= 1e-12


def test_sharded_and_adaptive_runs():
    text = EC.format(assign="").replace("QUBITS 5", "QUBITS 12")
    e1 = q.asm_run(text, seed=2)
    e4 = q.asm_run(text, ngpus=4, seed=2)
    assert e1["outcomes"] == e4["outcomes"]
    assert np.max(np.abs(e1["tables"] - e4["tables"])) <= 1e-12
    a1 = q.asm_run(text, encoding=q.ENC_ADAPTIVE2, seed=2)
    assert a1["outcomes"] == e1["outcomes"]
    assert np.max(np.abs(a1["tables"] - e1["tables"])) <= 0.011  # "about 3 digits"


def test_depolarizing_channel_at_px_1_is_an_x_after_every_gate():
    body = "H 0\nCNOT 0 1\nT 1\nU 1 2 3\nBEGIN MEASUREMENT\n"
    got = q.asm_run("QUBITS 4\nDEPOLARIZING CHANNEL P_X = 1\n" + body)
    explicit = "QUBITS 4\n" + "".join(f"{g}\n" + "".join(f"X {j}\n" for j in range(4))
                                      for g in body.splitlines() if g and not g.startswith("BEGIN")) + \
        "BEGIN MEASUREMENT\n"
    ref = q.asm_run(explicit)
    assert np.max(np.abs(got["tables"] - ref["tables"])) <= 1e-12
    # p = 0 channel == no channel; a weak channel changes something only by chance, but is reproducible
    none = q.asm_run("QUBITS 4\n" + body)
    zero = q.asm_run("QUBITS 4\nDEPOLARIZING CHANNEL P_X = 0, SEED = 3\n" + body)
    assert np.max(np.abs(none["tables"] - zero["tables"])) == 0.0
    w1 = q.asm_run("QUBITS 4\nDEPOLARIZING CHANNEL P_X = 0.3, P_Z = 0.3, SEED = 11\n" + body)
    w2 = q.asm_run("QUBITS 4\nDEPOLARIZING CHANNEL P_X = 0.3, P_Z = 0.3, SEED = 11\n" + body)
    assert np.array_equal(w1["tables"], w2["tables"])


def test_exit_measures_every_qubit_and_stops():
    got = q.asm_run("QUBITS 3\nX 1\nEXIT\nBEGIN MEASUREMENT\n", seed=1)
    assert got["outcomes"] == [(0, 0), (1, 1), (2, 0)]
    assert len(got["tables"]) == 0
