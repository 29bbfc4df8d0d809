"""World-size-2 CPU test (gloo) of the sharded path's host logic (SURVEY.md
§8(a) a7, §8(e)): two processes, one shard each, follow the library's own plan
(qsim_plan: the host planner compiled into libqsim.so, no GPU needed) and
perform every EXCHANGE exactly as the NCCL pipeline in api.cu does -- partner
r ^ 2^(g-nl), each rank sends its slot(l = 1-b) half chunk by chunk and the
received chunk lands in slot(l = 1-b) -- then apply the gate records on their
local amplitudes (global controls as rank-bit predicates, diagonal gates on
global bits as uniform factors).  The gathered state must equal the oracle's.
The per-shard arithmetic here is numpy test scaffolding; on the GPU the same
plan is executed by the CUDA kernels (tests/test_gpu_e.py loopback tests)."""
import os
import socket

import numpy as np
import pytest

import qsim_inputs as C

q = pytest.importorskip("paper_1805_04708_b200")
torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ins0(w, p):
    return ((w >> p) << (p + 1)) | (w & ((1 << p) - 1))


def _worker(rank, world, port, n, seed, chunk, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # plumbing used by bench.py for the NCCL unique id: an object broadcast from rank 0
        obj = [b"x" * 128 if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == b"x" * 128
        circ = _circuit(n, world, seed)
        ops, fmap = q.qsim_plan(n, world, circ)
        k = int(np.log2(world))
        nl = n - k
        a = np.zeros(1 << nl, dtype=np.complex128)
        if rank == 0:
            a[0] = 1
        idx = np.arange(1 << nl)
        nex = 0
        # phi[r]: physical global bits held by rank r (permuted by QSIM_OP_RELABEL)
        phi = list(range(world))
        nrm = 0
        i = 0
        while i < len(ops):
            o = ops[i]
            i += 1
            if o["type"] == q.OP_REMAP:
                # one all-to-all (api.cu remap): gather the group, blocks by the sorted local bits
                grp = [o]
                while i < len(ops) and ops[i]["type"] == q.OP_REMAP and ops[i]["gate_index"] == o["gate_index"]:
                    grp.append(ops[i])
                    i += 1
                grp.sort(key=lambda x: x["l"])
                m = len(grp)
                pos = [x["l"] for x in grp]
                jb = [x["g"] - nl for x in grp]
                ta = sum(((phi[rank] >> jb[b]) & 1) << b for b in range(m))

                def with_j(ph, t):
                    for b in range(m):
                        ph = (ph & ~(1 << jb[b])) | (((t >> b) & 1) << jb[b])
                    return ph

                def block_index(x, t):  # x-th index of block t (block bits inserted in ascending order)
                    w = x
                    for b in range(m):
                        w = _ins0(w, pos[b]) | (((t >> b) & 1) << pos[b])
                    return w

                nblock = 1 << (nl - m)
                C_ = 1
                while C_ * 2 * ((1 << m) - 1) <= chunk and C_ * 2 <= nblock:
                    C_ *= 2
                for c in range(nblock // C_):
                    xs = np.arange(c * C_, (c + 1) * C_)
                    reqs, recvs = [], []
                    for t in range(1 << m):
                        if t == ta:
                            continue
                        peer = phi.index(with_j(phi[rank], t))
                        send = torch.from_numpy(a[block_index(xs, t)].copy())
                        recv = torch.empty_like(send)
                        reqs += [dist.isend(send, peer), dist.irecv(recv, peer)]
                        recvs.append((t, recv))
                    for r in reqs:
                        r.wait()
                    for t, recv in recvs:
                        a[block_index(xs, t)] = recv.numpy()
                nrm += 1
                nex += 1
                continue
            if o["type"] == q.OP_RELABEL:
                _, kind, t, t2, ctl, u = circ.gate(o["gate_index"])
                jt = o["l"] - nl
                on = [all((phi[r] >> (c - nl)) & 1 for c in o["controls"]) for r in range(world)]
                if on[rank]:  # phase part diag(u10, u01) on the global target: a factor on the shard
                    a *= u[0, 1] if (phi[rank] >> jt) & 1 else u[1, 0]
                phi = [phi[r] ^ (1 << jt) if on[r] else phi[r] for r in range(world)]
                continue
            if o["type"] == q.OP_EXCHANGE:
                g, l = o["g"], o["l"]
                j = g - nl
                b = (phi[rank] >> j) & 1
                partner = phi.index(phi[rank] ^ (1 << j))
                half = 1 << (nl - 1)
                C_ = min(chunk, half, 1 << l)
                for c in range(half // C_):
                    start = _ins0(c * C_, l) + ((1 - b) << l)  # slot(l = 1-b), contiguous run
                    send = torch.from_numpy(a[start:start + C_].copy())
                    recv = torch.empty_like(send)
                    reqs = [dist.isend(send, partner), dist.irecv(recv, partner)]
                    for r in reqs:
                        r.wait()
                    a[start:start + C_] = recv.numpy()
                nex += 1
                continue
            _, kind, t, t2, ctl, u = circ.gate(o["gate_index"])
            pt = o["l"]
            ok = all(((phi[rank] >> (c - nl)) & 1) for c in o["controls"] if c >= nl)
            if not ok:
                continue
            cm = 0
            for c in o["controls"]:
                if c < nl:
                    cm |= 1 << c
            if pt >= nl:  # diagonal gate on a global bit: uniform factor on the shard
                assert o["cls"] == 1
                f = u[1, 1] if (phi[rank] >> (pt - nl)) & 1 else u[0, 0]
                sel = (idx & cm) == cm
                a[sel] *= f
                continue
            sel = (((idx >> pt) & 1) == 0) & ((idx & cm) == cm)
            i0 = idx[sel]
            i1 = i0 | (1 << pt)
            x, y = a[i0].copy(), a[i1].copy()
            a[i0] = u[0, 0] * x + u[0, 1] * y
            a[i1] = u[1, 0] * x + u[1, 1] * y
        # gather in logical order on rank 0
        full = [torch.zeros(1 << nl, dtype=torch.complex128) for _ in range(world)]
        dist.all_gather(full, torch.from_numpy(a))
        if rank == 0:
            blocks = [None] * world
            for r in range(world):
                blocks[phi[r]] = full[r].numpy()  # rank r holds physical global bits phi[r]
            phys = np.concatenate(blocks)
            pidx = np.arange(1 << n)
            L = np.zeros(1 << n, dtype=np.int64)
            for qq in range(n):
                L |= ((pidx >> fmap[qq]) & 1) << qq
            logical = np.empty_like(phys)
            logical[L] = phys
            out_q.put((logical, nex))
    finally:
        dist.destroy_process_group()


def _circuit(n, world, seed):
    circ = C.global_permutations(n, world, seed)
    circ.extend(C.config(0, n=n, seed=seed))
    circ.extend(C.layered(n, 2, seed=seed, h_first=False))
    circ.swap(1, n - 1)
    circ.extend(C.global_permutations(n, world, seed + 1))
    return circ


@pytest.mark.parametrize("chunk", [1 << 30, 32])
def test_four_rank_remap_protocol_matches_oracle(chunk):
    """World size 4 (2 global bits): the layered part needs both global
    qubits, so the plan holds all-to-all remaps (NEXT-1 (i)); every rank
    trades its 3 foreign blocks with the 3 partners chunk by chunk as the
    NCCL path in api.cu does (pack -> grouped send/recv -> unpack)."""
    import oracle

    n, seed, world = 11, 5, 4
    ops, _ = q.qsim_plan(n, world, _circuit(n, world, seed))
    assert sum(o["type"] == q.OP_REMAP for o in ops) >= 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, seed, chunk, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    logical, nex = out_q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ref = oracle.e_simulate(n, _circuit(n, world, seed))
    assert nex > 0
    assert np.max(np.abs(logical - ref)) <= 1e-12


@pytest.mark.parametrize("chunk", [1 << 30, 64])
def test_two_rank_exchange_protocol_matches_oracle(chunk):
    import oracle

    n, seed, world = 11, 3, 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, seed, chunk, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    logical, nex = out_q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    circ = _circuit(n, world, seed)
    ref = oracle.e_simulate(n, circ)
    assert nex > 0
    assert np.max(np.abs(logical - ref)) <= 1e-12
