"""qsim_inputs -- seeded synthetic circuit generators: the ONLY module shared by the oracle
side (tests / bench cpu_baseline) and the CUDA side.

It holds no arithmetic of the method (no state update, no encoding, no
reduction): it only builds gate *records* -- target, controls and the explicit
2x2 complex matrix of each gate -- from the gate definitions of PAPER.md App. B
 and from seeded random draws
(``numpy.random.Generator(PCG64(seed))``).  Both sides consume the identical
records, so no random draw is ever recomputed on either side.

Gate record layout (``Circuit`` arrays, one entry per gate):
  kind[g]    0 = controlled 2x2 gate, 1 = SWAP(target, target2)
  target[g]  target qubit
  target2[g] second qubit of a SWAP, else -1
  nctrl[g]   number of controls (0..2)
  ctrl[2g:2g+2]  control qubits (unused slots = -1)
  u[8g:8g+8] U row-major interleaved {u00r,u00i,u01r,u01i,u10r,u10i,u11r,u11i};
             row = output |0>,|1> of the target; applied iff all controls are 1.

Workload recipes follow SURVEY.md §8(d) (BASELINE.json configs 1-5).
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

SQ2 = 1.0 / math.sqrt(2.0)

# --- App. B gate matrices and reading A13 (Rz, Rx, CPHASE)


def mat_I():
    return np.eye(2, dtype=np.complex128)


def mat_H():
    return SQ2 * np.array([[1, 1], [1, -1]], dtype=np.complex128)


def mat_X():
    return np.array([[0, 1], [1, 0]], dtype=np.complex128)


def mat_Y():
    return np.array([[0, -1j], [1j, 0]], dtype=np.complex128)


def mat_Z():
    return np.array([[1, 0], [0, -1]], dtype=np.complex128)


def mat_S(dagger=False):
    return np.array([[1, 0], [0, -1j if dagger else 1j]], dtype=np.complex128)


def mat_T(dagger=False):
    return np.array([[1, 0], [0, (1 - 1j) * SQ2 if dagger else (1 + 1j) * SQ2]], dtype=np.complex128)


def mat_U1(lam):
    return np.array([[1, 0], [0, np.exp(1j * lam)]], dtype=np.complex128)


def mat_U2(phi, lam):
    return SQ2 * np.array([[1, -np.exp(1j * lam)], [np.exp(1j * phi), np.exp(1j * (phi + lam))]], dtype=np.complex128)


def mat_U3(theta, phi, lam):
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    return np.array([[c, -np.exp(1j * lam) * s], [np.exp(1j * phi) * s, np.exp(1j * (phi + lam)) * c]],
                    dtype=np.complex128)


def mat_pX(sign=+1):  # +X / -X
    return SQ2 * np.array([[1, sign * 1j], [sign * 1j, 1]], dtype=np.complex128)


def mat_pY(sign=+1):  # +Y / -Y
    return SQ2 * np.array([[1, sign * 1], [-sign * 1, 1]], dtype=np.complex128)


def mat_R(k):  # R(k) / R^dagger(k) for negative k, PAPER.md:1284, 1294 (reading A16)
    if k == 0:
        return mat_I()
    sgn = 1 if k > 0 else -1
    return np.array([[1, 0], [0, np.exp(sgn * 2j * math.pi / 2 ** abs(k))]], dtype=np.complex128)


def mat_Rz(theta):  # reading A13
    return np.array([[np.exp(-0.5j * theta), 0], [0, np.exp(0.5j * theta)]], dtype=np.complex128)


def mat_Rx(theta):  # reading A13 (+X = Rx(-pi/2))
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)


def mat_haar(rng: np.random.Generator):
    """Haar-random U(2): QR of a complex Ginibre matrix, columns rescaled by the
    phases of diag(R) (Mezzadri's method; reading A13)."""
    z = (rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))) / math.sqrt(2.0)
    q, r = np.linalg.qr(z)
    d = np.diagonal(r)
    return q * (d / np.abs(d))[None, :]


# --- circuit container


@dataclass
class Circuit:
    n: int
    names: list = field(default_factory=list)
    _kind: list = field(default_factory=list)
    _target: list = field(default_factory=list)
    _target2: list = field(default_factory=list)
    _nctrl: list = field(default_factory=list)
    _ctrl: list = field(default_factory=list)
    _u: list = field(default_factory=list)
    _frozen: dict = field(default_factory=dict)

    def add(self, name, u, target, controls=()):
        assert 0 <= target < self.n and len(controls) <= 2
        assert target not in controls and len(set(controls)) == len(controls)
        for c in controls:
            assert 0 <= c < self.n
        self.names.append(name)
        self._kind.append(0)
        self._target.append(int(target))
        self._target2.append(-1)
        self._nctrl.append(len(controls))
        self._ctrl.append([int(c) for c in controls] + [-1] * (2 - len(controls)))
        self._u.append(np.asarray(u, dtype=np.complex128).reshape(2, 2))
        self._frozen.clear()
        return self

    def swap(self, q1, q2):
        assert q1 != q2 and 0 <= q1 < self.n and 0 <= q2 < self.n
        self.names.append("SWAP")
        self._kind.append(1)
        self._target.append(int(q1))
        self._target2.append(int(q2))
        self._nctrl.append(0)
        self._ctrl.append([-1, -1])
        self._u.append(mat_I())
        self._frozen.clear()
        return self

    def extend(self, other: "Circuit"):
        assert other.n == self.n
        for i in range(len(other)):
            if other._kind[i] == 1:
                self.swap(other._target[i], other._target2[i])
            else:
                ctl = [c for c in other._ctrl[i] if c >= 0]
                self.add(other.names[i], other._u[i], other._target[i], ctl)
        return self

    def __len__(self):
        return len(self._kind)

    def _arr(self, key):
        if not self._frozen:
            self._frozen["kind"] = np.asarray(self._kind, dtype=np.int32)
            self._frozen["target"] = np.asarray(self._target, dtype=np.int32)
            self._frozen["target2"] = np.asarray(self._target2, dtype=np.int32)
            self._frozen["nctrl"] = np.asarray(self._nctrl, dtype=np.int32)
            self._frozen["ctrl"] = np.asarray(self._ctrl, dtype=np.int32).reshape(-1)
            u = np.stack(self._u) if self._u else np.zeros((0, 2, 2), np.complex128)
            self._frozen["u"] = np.ascontiguousarray(u).view(np.float64).reshape(-1)
        return self._frozen[key]

    kind = property(lambda s: s._arr("kind"))
    target = property(lambda s: s._arr("target"))
    target2 = property(lambda s: s._arr("target2"))
    nctrl = property(lambda s: s._arr("nctrl"))
    ctrl = property(lambda s: s._arr("ctrl"))
    u = property(lambda s: s._arr("u"))

    def gate(self, i):
        """(name, kind, target, target2, controls, U 2x2) of gate i."""
        ctl = tuple(c for c in self._ctrl[i] if c >= 0)
        return self.names[i], self._kind[i], self._target[i], self._target2[i], ctl, self._u[i]

    def slice(self, start, stop):
        c = Circuit(self.n)
        for i in range(start, stop):
            name, kind, t, t2, ctl, u = self.gate(i)
            if kind == 1:
                c.swap(t, t2)
            else:
                c.add(name, u, t, ctl)
        return c


# --- workloads (BASELINE.json configs)

CFG1_KINDS = ("H", "X", "Y", "Z", "S", "T", "Rz", "Rx", "Haar", "CNOT", "CPHASE", "TOFFOLI")


def random_circuit(n: int = 14, ngates: int = 200, seed: int = 0, kinds=CFG1_KINDS) -> Circuit:
    """Config 1: kind uniform over ``kinds``; qubits drawn uniformly without
    replacement (controls first, then target); angles ~ U[0, 2pi)."""
    rng = np.random.default_rng(seed)
    c = Circuit(n)
    for _ in range(ngates):
        k = kinds[rng.integers(len(kinds))]
        nq = {"CNOT": 2, "CPHASE": 2, "TOFFOLI": 3}.get(k, 1)
        q = [int(x) for x in rng.choice(n, size=nq, replace=False)]
        ctl, t = q[:-1], q[-1]
        if k == "H":
            c.add(k, mat_H(), t)
        elif k == "X":
            c.add(k, mat_X(), t)
        elif k == "Y":
            c.add(k, mat_Y(), t)
        elif k == "Z":
            c.add(k, mat_Z(), t)
        elif k == "S":
            c.add(k, mat_S(), t)
        elif k == "T":
            c.add(k, mat_T(), t)
        elif k == "Rz":
            c.add(k, mat_Rz(rng.uniform(0, 2 * math.pi)), t)
        elif k == "Rx":
            c.add(k, mat_Rx(rng.uniform(0, 2 * math.pi)), t)
        elif k == "Haar":
            c.add(k, mat_haar(rng), t)
        elif k == "CNOT":
            c.add(k, mat_X(), t, ctl)
        elif k == "CPHASE":
            c.add(k, mat_U1(rng.uniform(0, 2 * math.pi)), t, ctl)
        elif k == "TOFFOLI":
            c.add(k, mat_X(), t, ctl)
        else:
            raise ValueError(k)
    return c


def global_permutations(n: int, nshards: int, seed: int) -> Circuit:
    """Permutation gates whose target and controls are all among the top
    log2(nshards) qubits (the global qubits of a fresh state): X, Y, and, when
    there are enough global qubits, CNOT and Toffoli (App. B, PAPER.md:1141,
    1151, 1300-1363), each after an H on a random local qubit so the state is
    not a basis state.  Seeded (PCG64)."""
    rng = np.random.default_rng(seed)
    k = int(round(np.log2(nshards)))
    top = list(range(n - k, n))
    c = Circuit(n)
    for _ in range(6):
        c.add("H", mat_H(), int(rng.integers(0, n - k)))
        kind = int(rng.integers(0, 4))
        perm = [int(q) for q in rng.permutation(top)]
        if kind == 0 or k == 1 and kind >= 2:
            c.add("X", mat_X(), perm[0])
        elif kind == 1:
            c.add("Y", mat_Y(), perm[0])
        elif kind == 2 or k == 2:
            c.add("CNOT", mat_X(), perm[0], [perm[1]])
        else:
            c.add("TOFFOLI", mat_X(), perm[0], [perm[1], perm[2]])
    return c


def h_wall(n: int) -> Circuit:
    """PAPER.md §5.1 (653-657): H on every qubit of |0...0>."""
    c = Circuit(n)
    for q in range(n):
        c.add("H", mat_H(), q)
    return c


def ghz_chain(n: int) -> Circuit:
    """PAPER.md §5.2 (743-745): H 0; CNOT 0 1; ...; CNOT N-2 N-1."""
    c = Circuit(n)
    c.add("H", mat_H(), 0)
    for q in range(n - 1):
        c.add("CNOT", mat_X(), q + 1, [q])
    return c


def layered(n: int, layers: int, seed: int, entangle: bool = True, h_first: bool = True) -> Circuit:
    """Configs 2/3: H on all n, then ``layers`` x (Haar U(2) on every qubit
    0..n-1 in index order, then CNOTs on a random perfect matching: a random
    permutation p, CNOT p0->p1, p2->p3, ...).  ``entangle=False`` drops the
    CNOTs (product-state pin, Eq. appa2) while keeping the same U(2) draws."""
    rng = np.random.default_rng(seed)
    c = Circuit(n)
    if h_first:
        for q in range(n):
            c.add("H", mat_H(), q)
    for _ in range(layers):
        for q in range(n):
            c.add("Haar", mat_haar(rng), q)
        perm = rng.permutation(n)
        for i in range(0, n - 1, 2):
            if entangle:
                c.add("CNOT", mat_X(), int(perm[i + 1]), [int(perm[i])])
    return c


def rz_rx_cphase(n: int, layers: int, seed: int) -> Circuit:
    """Config 4: H on all, then ``layers`` x (per qubit a coin flip picks Rz(theta)
    or Rx(theta), theta ~ U[0,2pi); then CPHASE(phi ~ U[0,2pi)) on a random
    perfect matching)."""
    rng = np.random.default_rng(seed)
    c = Circuit(n)
    for q in range(n):
        c.add("H", mat_H(), q)
    for _ in range(layers):
        for q in range(n):
            th = rng.uniform(0, 2 * math.pi)
            if rng.integers(2):
                c.add("Rx", mat_Rx(th), q)
            else:
                c.add("Rz", mat_Rz(th), q)
        perm = rng.permutation(n)
        for i in range(0, n - 1, 2):
            c.add("CPHASE", mat_U1(rng.uniform(0, 2 * math.pi)), int(perm[i + 1]), [int(perm[i])])
    return c


def qft(n: int, x: int | None = None, seed: int = 5) -> tuple[Circuit, int]:
    """Config 5 (reading A15): X on the set bits of x, then for j = n-1..0
    { H(j); for m = j-1..0: CPHASE(control m, target j, 2pi/2^(j-m+1)) },
    then SWAP(i, n-1-i) for i < n/2.  Returns (circuit, x)."""
    if x is None:
        x = int(np.random.default_rng(seed).integers(0, 1 << n, dtype=np.uint64))
    c = Circuit(n)
    for q in range(n):
        if (x >> q) & 1:
            c.add("X", mat_X(), q)
    for j in range(n - 1, -1, -1):
        c.add("H", mat_H(), j)
        for m in range(j - 1, -1, -1):
            c.add("CPHASE", mat_R(j - m + 1), j, [m])
    for i in range(n // 2):
        c.swap(i, n - 1 - i)
    return c, x


def qft_register(n: int, m: int, swaps: bool = True) -> Circuit:
    """The QFT of reading A15 on qubits 0..m-1 of an n-qubit register (no input
    preparation): for j = m-1..0 { H(j); CPHASE(k -> j, 2pi/2^(j-k+1)), k = j-1..0 },
    then (if swaps) SWAP(i, m-1-i) for i < m/2."""
    c = Circuit(n)
    for j in range(m - 1, -1, -1):
        c.add("H", mat_H(), j)
        for k in range(j - 1, -1, -1):
            c.add("CPHASE", mat_R(j - k + 1), j, [k])
    if swaps:
        for i in range(m // 2):
            c.swap(i, m - 1 - i)
    return c


def draper_adder(k: int, a: int, b: int) -> Circuit:
    """The QFT adder of PAPER.md section 5.3 (Table 4; Draper's
    construction, DRAP00) on n = 2k qubits: b on qubits 0..k-1 (bit j on qubit
    j), a on qubits k..2k-1 in reversed bit order (bit j of a on qubit 2k-1-j:
    the layout Table 4's a-register column shows, reading R-B12).  X gates
    prepare |b>|a>; QFT without swaps on the b register (reading A15: for
    j = k-1..0 { H(j); CPHASE(m -> j, 2pi/2^(j-m+1)), m = j-1..0 }) gives qubit
    j the phase 2pi (b mod 2^(j+1))/2^(j+1); CPHASE(a_m -> j, 2pi/2^(j-m+1)),
    m <= j, adds a's; the inverse QFT returns |a + b mod 2^k> on qubits 0..k-1.
    Gate count: popcount(a) + popcount(b) + 3 k (k + 1)/2."""
    n = 2 * k
    c = Circuit(n)
    for j in range(k):
        if (b >> j) & 1:
            c.add("X", mat_X(), j)
        if (a >> j) & 1:
            c.add("X", mat_X(), n - 1 - j)
    for j in range(k - 1, -1, -1):
        c.add("H", mat_H(), j)
        for m in range(j - 1, -1, -1):
            c.add("CPHASE", mat_R(j - m + 1), j, [m])
    for j in range(k - 1, -1, -1):
        for m in range(j, -1, -1):
            c.add("CPHASE", mat_R(j - m + 1), j, [n - 1 - m])
    for j in range(k):
        for m in range(j):
            c.add("CPHASE", mat_R(-(j - m + 1)), j, [m])
        c.add("H", mat_H(), j)
    return c


def config(idx: int, n: int | None = None, seed: int | None = None, layers: int | None = None) -> Circuit:
    """BASELINE.json configs by index (0-based as in the JSON list)."""
    if idx == 0:
        return random_circuit(14 if n is None else n, 200, 0 if seed is None else seed)
    if idx == 1:
        return layered(30 if n is None else n, 20 if layers is None else layers, 1 if seed is None else seed)
    if idx == 2:
        return layered(36 if n is None else n, 10 if layers is None else layers, 3 if seed is None else seed)
    if idx == 3:
        return rz_rx_cphase(39 if n is None else n, 10 if layers is None else layers, 4 if seed is None else seed)
    if idx == 4:
        return qft(35 if n is None else n, seed=5 if seed is None else seed)[0]
    raise ValueError(idx)


def random_codes(n: int, seed: int, frac_zero: float = 0.05, frac_one: float = 0.0):
    """Seeded random A-variant codes (b0, b1 int8 interleaved) plus bounds
    0 < r0 < r1 < 1 -- synthetic inputs for per-gate A parity tests."""
    rng = np.random.default_rng(seed)
    dim = 1 << n
    b0 = rng.integers(-127, 127, size=dim, dtype=np.int16)
    b1 = rng.integers(-128, 128, size=dim, dtype=np.int16)
    u = rng.random(dim)
    b0[u < frac_zero] = -128
    b0[(u >= frac_zero) & (u < frac_zero + frac_one)] = 127
    codes = np.empty(2 * dim, dtype=np.int8)
    codes[0::2] = b0.astype(np.int8)
    codes[1::2] = b1.astype(np.int8)
    r0 = float(rng.uniform(0.05, 0.2)) * 2.0 ** (-n / 2)
    r1 = r0 + float(rng.uniform(1.0, 4.0)) * 2.0 ** (-n / 2)
    return codes, r0, r1


def splitmix_uniform(seed: int, count: int) -> np.ndarray:
    """The counter-based draws of qsim_measure / qsim_sample (include/qsim.h):
    u_k = (splitmix64(seed + k) >> 11) * 2^-53, k = 0..count-1.  Both the CUDA
    side and the oracle side use exactly these numbers."""
    M = (1 << 64) - 1
    out = np.empty(count, dtype=np.float64)
    for i in range(count):
        x = (seed + i + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        x ^= x >> 31
        out[i] = (x >> 11) * (1.0 / 9007199254740992.0)
    return out
