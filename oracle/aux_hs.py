"""ORACLE -- test infrastructure only (see oracle/__init__.py).

The auxiliary-variable method of PAPER.md §4.2 (lines 462-591), followed step
by step in the paper's notation, in plain numpy fp64/complex128:

1. Every CNOT_{c t} is rewritten as H_t U_{c t}(pi) H_t.
   Reading R-B9 (the paper names single-qubit gates, controlled phase shifts
   and CNOT): a controlled diagonal gate diag(d0, d1) on t with
   control c is diag(1, d0) on c followed by U_{c t}(a), e^{ia} = d1 / d0
   (d0 != 0; no variable when d1 = d0, U_ct(0) = I, so a CNOT or a
   controlled phase costs exactly one variable); a controlled
   anti-diagonal [[0, u01], [u10, 0]] is the
   controlled diagonal diag(u10, u01) followed by CNOT_{c t}.  Gates with two
   controls or a controlled dense 2x2 are outside the method (ValueError).
2. Each U_{c t}(a_p) (Eq. appa4) gets an auxiliary variable
   s_p = +-1 and the discrete Hubbard-Stratonovich identity (Eqs. appa5-appa6,
   P:560-575)
       U_{ct}(a) = 1/2 sum_{s=+-1} exp(i (sigma^z_c + sigma^z_t)(x s - a/4)),
       cos 2x = exp(i a / 2)   (x complex; principal arccos),
   i.e. on qubit c and on qubit t the single-qubit diagonal
   diag(e^{i(x s - a/4)}, e^{-i(x s - a/4)})  (sigma^z = +1 on |0>).
3. For every assignment (s_1..s_P), W_j(s) is the product, in circuit order,
   of qubit j's single-qubit operations (Eq. appa1), and
       <y|psi> = 2^{-P} sum_s prod_j <y_j| W_j(s) |0>_j     (Eq. appa7).

No blocking or reordering beyond the definitions above; the assignments are
enumerated as s_p = +1 if bit p of the counter is 0, -1 otherwise.
"""
from __future__ import annotations

import numpy as np


def _rewrite(circuit):
    """Step 1: the circuit as a list of ('u', j, 2x2) and ('cp', c, t, a) ops."""
    ops = []
    for g in range(len(circuit)):
        name, kind, t, t2, ctl, u = circuit.gate(g)
        if kind == 1:
            raise ValueError("SWAP is outside the auxiliary-variable method")
        u = np.asarray(u, dtype=np.complex128)
        if len(ctl) == 0:
            ops.append(("u", t, u))
            continue
        if len(ctl) > 1:
            raise ValueError("gates with two controls are outside the method (P:470-472)")
        c = ctl[0]
        diag = u[0, 1] == 0 and u[1, 0] == 0
        anti = u[0, 0] == 0 and u[1, 1] == 0
        if diag:
            d0, d1 = u[0, 0], u[1, 1]
            ops.append(("u", c, np.diag([1.0, d0])))
            if d1 != d0:  # U_ct(0) = I needs no variable
                ops.append(("cp", c, t, float(np.angle(d1 / d0))))
        elif anti:
            d0, d1 = u[1, 0], u[0, 1]  # U = X diag(u10, u01)
            ops.append(("u", c, np.diag([1.0, d0])))
            if d1 != d0:
                ops.append(("cp", c, t, float(np.angle(d1 / d0))))
            h = np.array([[1, 1], [1, -1]], dtype=np.complex128) / np.sqrt(2.0)
            ops.append(("u", t, h))
            ops.append(("cp", c, t, np.pi))
            ops.append(("u", t, h))
        else:
            raise ValueError("controlled dense 2x2 is outside the method (P:470-472)")
    return ops


def num_aux(circuit) -> int:
    return sum(1 for o in _rewrite(circuit) if o[0] == "cp")


def amplitudes(n: int, circuit, idx, return_abs_sum: bool = False):
    """<y|psi> for every logical index y in idx by Eq. appa7.  With
    return_abs_sum, also 2^{-P} sum_s |prod_j ...| (the size of the terms that
    cancel in the sum -- the scale of its rounding error)."""
    ops = _rewrite(circuit)
    cps = [o for o in ops if o[0] == "cp"]
    P = len(cps)
    ns = 1 << P
    cnt = np.arange(ns, dtype=np.int64)
    # step 2: x_p with cos 2x_p = e^{i a_p / 2}
    xs = [np.arccos(np.exp(0.5j * a)) / 2.0 for (_, _, _, a) in cps]
    # step 3: W_j(s)|0> for all s at once, qubit by qubit, ops in circuit order
    vec = np.zeros((n, ns, 2), dtype=np.complex128)
    vec[:, :, 0] = 1.0
    p = 0
    for o in ops:
        if o[0] == "u":
            _, j, u = o
            vec[j] = vec[j] @ u.T
        else:
            _, c, t, a = o
            s = np.where((cnt >> p) & 1, -1.0, 1.0)
            th = xs[p] * s - a / 4.0
            for j in (c, t):
                vec[j, :, 0] *= np.exp(1j * th)
                vec[j, :, 1] *= np.exp(-1j * th)
            p += 1
    idx = np.asarray(idx, dtype=np.int64)
    out = np.empty(len(idx), dtype=np.complex128)
    absum = np.empty(len(idx))
    for k, y in enumerate(idx):
        prod = np.ones(ns, dtype=np.complex128)
        for j in range(n):
            prod *= vec[j, :, (int(y) >> j) & 1]
        out[k] = prod.sum() / ns
        absum[k] = np.abs(prod).sum() / ns
    return (out, absum) if return_abs_sum else out
