"""One process driving P GPUs (QSIM_TRANSPORT_DEVICES, the qsim_create(N, enc,
ngpus) process model of SURVEY.md §8(e)): member r of the
handle owns shard r on device r, an in-process NCCL communicator carries the
exchanges, one host thread per device runs each call.  With one visible GPU
the group runs with P = 1 (threads, dispatch and the NCCL read-out paths);
P = 2 runs when two GPUs are visible (the driver's 1-GPU boxes skip it)."""
import numpy as np
import pytest

import oracle
import qsim_inputs as C

pytestmark = pytest.mark.gpu
q = pytest.importorskip("paper_1805_04708_b200")
torch = pytest.importorskip("torch")
TOL = 1e-12


def ndev():
    return torch.cuda.device_count()


@pytest.mark.parametrize("enc", [0, 1])
def test_device_group_of_one(enc):
    n = 14
    circ = C.config(0, seed=3)
    with q.State(n, enc, 1, transport=q.TRANSPORT_DEVICES, device=0) as s:
        s.apply_circuit(circ)
        z = s.get_state()
        ex = s.expectations()
        st = s.stats()
        p1 = s.probabilities()
        nrm = s.norm()
        amps = s.get_amplitudes(np.array([0, 5, 1 << 13], dtype=np.uint64))
    if enc == 0:
        ref = oracle.e_simulate(n, circ)
        assert np.max(np.abs(z - ref)) <= TOL
    else:  # A: the same codes as the one-device handle (the oracle-A parity is test_gpu_a*.py's)
        with q.State(n, enc) as one:
            one.apply_circuit(circ)
            assert np.array_equal(z, one.get_state())
    assert np.max(np.abs(ex - oracle.e_expectations(z, n))) <= TOL
    assert np.max(np.abs(p1 - ex[:, 2] * nrm)) <= TOL
    assert np.max(np.abs(amps - z[[0, 5, 1 << 13]])) <= 1e-15
    assert st["kernels"] > 0 and st["gates"] == len(circ)


def test_qsim_create_spans_devices():
    """qsim_create(N, enc, ngpus) asks for ngpus devices: EINVAL (with the
    device count in the message) when fewer are visible."""
    if ndev() >= 2:
        pytest.skip("two devices visible: covered by test_two_devices_vs_oracle")
    with pytest.raises(q.QsimError) as err:
        q.qsim_create(16, q.ENC_FP64, 2)
    assert err.value.code == -1 and "visible" in str(err.value)


@pytest.mark.skipif("torch.cuda.device_count() < 2")
@pytest.mark.parametrize("enc", [0, 1])
def test_two_devices_vs_oracle(enc):
    """P = 2 on devices 0 and 1 from one process: global-qubit gates exchange
    half a shard over NVLink; results equal the oracle (E 1e-12) / the
    single-GPU run bit for bit (A: exact global bounds)."""
    n = 16
    circ = C.layered(n, 3, seed=2)
    h = q.qsim_create(n, enc, 2)
    try:
        q.qsim_apply_circuit(h, circ)
        z = np.empty(1 << n, dtype=np.complex128)
        q._check(q._lib.qsim_get_state(h, q._dptr(z.view(np.float64))))
        ex = q.qsim_expectations(h, n)
        st = q.qsim_get_stats(h)
    finally:
        q.qsim_destroy(h)
    assert st["exchanges"] > 0
    if enc == 0:
        assert np.max(np.abs(z - oracle.e_simulate(n, circ))) <= TOL
    else:
        with q.State(n, enc) as one:
            one.apply_circuit(circ)
            assert np.array_equal(z, one.get_state())
    assert np.max(np.abs(ex - oracle.e_expectations(z, n))) <= TOL
