#!/usr/bin/env python
"""Benchmark of the JUQCS hot path on B200 (BASELINE.json metric).

Workload (one "step" = one pass of the whole hot path over one batch of
synthetic input = the whole circuit applied to the resident state):
  BASELINE config 3 at every P = 1/2/4/8 GPUs: N = 33 + log2(P) qubits, E
  fp64, 2^33 amplitudes (128 GiB) per GPU, top log2(P) qubits global; H on
  all N, then 10 layers of Haar U(2) on every qubit + CNOTs on a random
  perfect matching (seed 3; 523/544/555/576 gates).  P = 1 is the weak-scaling
  base point and the largest single-GPU E workload.  Launch: torchrun (one
  process per GPU, QSIM_TRANSPORT_NCCL) or plain `python bench.py --gpus P`
  (one process driving P GPUs, QSIM_TRANSPORT_DEVICES).
value = aggregate effective HBM GB/s = sum over gates of the gate's
algorithmic bytes (SURVEY.md §8(d) byte-accounting: 32 B x amplitudes touched
by the gate, 0 for SWAP) over all GPUs / device time (max over ranks).
Inputs are larger than L2 (128 GiB state >> 126 MB), so no L2 flush is needed.
Warm-up: the first warm-up step queues the NVRTC specialisation of every pass
program of the circuit; bench.py waits for them (qsim_jit_sync) before the
remaining warm-up steps, so the timed steps run the specialised pass kernels
(reported as library.jit_passes).

--impl reference: the oracle (plain CPU fp64 simulator, oracle/) timed on the
host cores on a bounded sample of the same workload, same metric and unit.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import qsim_inputs as C  # noqa: E402

METRIC = "gates/sec and effective HBM GB/s per gate sweep at N qubits, 1/2/4/8 B200"
ALU_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # fp64 FMA peak from unit counts and max clock
UNIT = "GB/s"


def gate_bytes(circ, amp_bytes=16) -> float:
    """Algorithmic bytes of every gate had it run alone."""
    n = circ.n
    tot = 0.0
    for g in range(len(circ)):
        name, kind, t, t2, ctl, u = circ.gate(g)
        if kind == 1:
            continue
        off = abs(u[0, 1]) == 0 and abs(u[1, 0]) == 0
        if off and u[0, 0] == 1 and u[1, 1] == 1:
            continue
        b = 2.0 * amp_bytes * 2.0 ** (n - len(ctl))
        if off and (u[0, 0] == 1 or u[1, 1] == 1):
            b *= 0.5
        tot += b
    return tot


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,memory.used,memory.total")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, mem, memtot, pw = [], None, set(), [], None, []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
            try:
                pw.append(float(parts[3]))
                mem.append(float(parts[8]))
                memtot = float(parts[9])
            except (ValueError, IndexError):
                pass
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
               "samples": len(sm)}
        if pw:
            out["power_w_median"] = statistics.median(pw)
        if mem:  # device memory in use during the timed region (the shard plus buffers fit)
            out["memory_used_gib_max"] = max(mem) / 1024.0
            out["memory_total_gib"] = memtot / 1024.0 if memtot else None
        return out


def workload(world):
    k = int(round(math.log2(world)))
    n = 33 + k
    circ = C.config(2, n=n)  # layered(n, 10, seed=3)
    name = (f"config3: N={n} E fp64, 2^33 amplitudes (128 GiB) per GPU, top {k} qubit(s) global, H wall + 10 layers "
            f"(Haar U(2) on every qubit + CNOT perfect matching), {len(circ)} gates, seed 3")
    return n, circ, name


def recipe(n):
    """The workload recipe at another size (the CPU legs' fallback when the host lacks the RAM)."""
    return C.config(2, n=n)


def cpu_sample(circ_full, budget_s=15.0):
    """Time the oracle on the first gates of the same workload (bounded sample)."""
    import oracle
    import psutil

    n = circ_full.n
    need = (16 << n) * 1.5
    if psutil.virtual_memory().available < need:
        n = 28
    circ = recipe(n) if n != circ_full.n else circ_full
    a = oracle.e_init(n)
    done, t_all, nbytes = 0, 0.0, 0.0
    while t_all < budget_s and done < len(circ):
        one = circ.slice(done, done + 1)
        t0 = time.perf_counter()
        oracle.e_run(a, n, one)
        t_all += time.perf_counter() - t0
        nbytes += gate_bytes(one)
        done += 1
    out = {"value": nbytes / t_all / 1e9, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
           "sample": f"first {done} gates of the workload's circuit at N={n} ({t_all:.1f} s, "
                     f"{done / t_all:.3f} gates/s)"}
    # the same oracle on one thread (1 thread and all cores), a short sample
    cores = oracle.num_threads()
    try:
        oracle.set_num_threads(1)
        done1, t1, b1 = 0, 0.0, 0.0
        while t1 < budget_s / 3 and done1 < len(circ):
            one = circ.slice(done1, done1 + 1)
            t0 = time.perf_counter()
            oracle.e_run(a, n, one)
            t1 += time.perf_counter() - t0
            b1 += gate_bytes(one)
            done1 += 1
        out["one_thread"] = {"value": b1 / t1 / 1e9, "unit": UNIT, "cores": 1,
                             "sample": f"first {done1} gates at N={n} ({t1:.1f} s)"}
    finally:
        oracle.set_num_threads(cores)
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    n, circ, name = workload(world)
    W, K = args.warmup, args.steps
    import oracle
    import psutil

    # torchrun sets OMP_NUM_THREADS=1 per rank; only rank 0 works here, so
    # the oracle gets every host core, as at N=1
    oracle.set_num_threads(len(os.sched_getaffinity(0)))
    if psutil.virtual_memory().available < (16 << n) * 1.5:
        n = 28
        circ = recipe(n)
    a = oracle.e_init(n)
    # each step: a bounded sample -- the next `g` gates of the circuit (about 2 s of CPU work)
    t0 = time.perf_counter()
    oracle.e_run(a, n, circ.slice(0, 1))
    t1 = max(time.perf_counter() - t0, 1e-3)
    g = max(1, int(2.0 / t1))
    pos = 1

    def step():
        nonlocal pos
        if pos + g > len(circ):
            pos = 0
        part = circ.slice(pos, pos + g)
        pos += g
        t0 = time.perf_counter()
        oracle.e_run(a, n, part)
        return time.perf_counter() - t0, gate_bytes(part), g

    for _ in range(W):
        step()
    tt, bb, gg = 0.0, 0.0, 0
    for _ in range(K):
        t, b, c = step()
        tt, bb, gg = tt + t, bb + b, gg + c
    v = bb / tt / 1e9
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": tt / K * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": name, "reference_sample": f"{g} gates per step at N={n}"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": f"{K} steps x {g} gates of the workload circuit at N={n}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gates_per_s": gg / tt}
    emit(line)
    return 0


# stdout carries exactly the one JSON line: everything else written to file
# descriptor 1 -- NCCL's version banner at communicator init, library or
# Python prints -- goes to stderr; the line is written to the saved stdout.
_OUT_FD = None


def emit(line: dict) -> None:
    data = (json.dumps(line) + "\n").encode()
    if _OUT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_OUT_FD, data)


def main():
    global _OUT_FD
    sys.stdout.flush()
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fuse", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-cold", action="store_true", help="skip the cold end-to-end leg")
    args = ap.parse_args()
    torchrun = "RANK" in os.environ and "WORLD_SIZE" in os.environ
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus))) if torchrun else args.gpus
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    assert args.warmup >= 3 or os.environ.get("BENCH_ALLOW_SHORT"), "timing rules: at least 3 warm-up steps"

    import torch

    torch.cuda.set_device(local)
    import paper_1805_04708_b200 as q

    dist = None
    # under torchrun: one process per GPU (NCCL transport); BENCH_FORCE_DIST=1
    # takes that path even with one rank (a one-GPU check of the plumbing).
    # Without torchrun, --gpus P > 1: this process drives P GPUs (DEVICES).
    use_dist = torchrun and (world > 1 or os.environ.get("BENCH_FORCE_DIST") == "1")
    if use_dist:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, circ, name = workload(world)
    if use_dist:
        obj = [q.qsim_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        s = q.State(n, q.ENC_FP64, world, transport=q.TRANSPORT_NCCL, rank=rank, device=local,
                    nccl_id=obj[0], fuse=args.fuse)
        devs = [local]
        mode = f"{world} processes (torchrun), one GPU each, NCCL exchange"
    elif world > 1:
        s = q.State(n, q.ENC_FP64, world, transport=q.TRANSPORT_DEVICES, device=0, fuse=args.fuse)
        devs = list(range(world))
        mode = f"one process driving {world} GPUs (QSIM_TRANSPORT_DEVICES), in-process NCCL exchange"
    else:
        s = q.State(n, q.ENC_FP64, 1, fuse=args.fuse, device=local)
        devs = [local]
        mode = "one GPU"
    gates = q.pack_gates(circ)  # host gate records (the step's input)
    # the library's stream on every device this process drives
    streams = [torch.cuda.ExternalStream(s.stream(r), device=torch.device("cuda", d)) for r, d in enumerate(devs)]

    def barrier():
        if dist:
            dist.barrier()

    def sync_all():
        for d in devs:
            torch.cuda.synchronize(d)

    for w in range(args.warmup):
        s.apply_circuit(gates)
        if w == 0:
            # the first step queued the run-time specialisation of every pass
            # program (NVRTC, background threads): wait for them so the later
            # warm-up steps and the timed region run the specialised kernels
            s.sync()
            q.qsim_jit_sync()
    s.sync()
    s.reset_stats()
    s.profile(True)
    s.profile_read()
    clocks = ClockSampler(local)
    clocks.start()
    evs = []
    for d in devs:
        with torch.cuda.device(d):
            evs.append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
    barrier()
    sync_all()
    s.sync()
    for (e0, _), st_ in zip(evs, streams):
        e0.record(st_)
    for _ in range(args.steps):
        s.apply_circuit(gates)
    for (_, e1), st_ in zip(evs, streams):
        e1.record(st_)
    s.sync()
    sync_all()
    barrier()
    clk = clocks.stop()
    ms = max(e0.elapsed_time(e1) for e0, e1 in evs)  # max over the devices this process drives
    st = s.stats()
    prof = s.profile_read()
    s.profile(False)
    t_dev = torch.tensor([ms, st["gate_bytes"], float(st["kernels"]), st["exchange_bytes"]], dtype=torch.float64,
                         device="cuda")
    if dist:
        mx = t_dev.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t_dev.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, bytes_all, launches, xbytes = mx[0].item(), sm[1].item(), int(sm[2].item()), sm[3].item()
    else:
        ms_max, bytes_all, launches, xbytes = ms, st["gate_bytes"], st["kernels"], st["exchange_bytes"]
    value = bytes_all / (ms_max / 1e3) / 1e9
    gates_per_s = len(circ) * args.steps / (ms_max / 1e3)

    # ---- exchange (a7): bytes sent per direction per GPU over the exchange time ----
    exchange = None
    if world > 1:
        xr = prof.get("xchg")
        per_gpu = xbytes / world
        if xr and xr["ms"] > 0:
            gbs = per_gpu / (xr["ms"] / 1e3) / 1e9
            exchange = {"GB_per_direction_per_gpu": per_gpu / 1e9, "exchange_ms": xr["ms"],
                        "GBps_per_direction": gbs, "frac_of_900": gbs / 900.0, "frac_of_measured_770": gbs / 770.0,
                        "what": "bytes each GPU sent (pairwise half-shard swaps + all-to-all remaps) / time of the "
                                "exchange launches (CUDA events on the library stream, rank 0)"}

    # ---- end to end through the public API with host buffers ----
    # every step: reset to |0...0> (the method's input state), H2D of the host
    # gate records, the circuit, D2H of the result (per-qubit probabilities).
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    sync_all()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        s.reset()
        s.apply_circuit(gates)
        p1 = s.probabilities()
    t_e2e = time.perf_counter() - t0
    barrier()
    if dist:
        tt = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = tt.item()
    e2e = {"value": bytes_all / args.steps * e2e_steps / t_e2e / 1e9, "unit": UNIT,
           "h2d_bytes_per_step": 88 * len(circ), "d2h_bytes_per_step": 8 * len(p1),
           "what": "qsim_reset + qsim_apply_circuit(host gate records) + qsim_probabilities(host buffer), wall clock"}

    # ---- cold end to end: a circuit never seen by this process every step ----
    # (fresh seed: new CNOT matchings and matrices, so the host plan cache
    # misses and the pass programs are new: planning + the interpreter while
    # NVRTC specialises in the background, or the on-disk cubin cache)
    if not args.no_cold:
        cold_steps = 2
        barrier()
        sync_all()
        t0 = time.perf_counter()
        cb = 0.0
        for i in range(cold_steps):
            c2 = C.layered(n, 10, seed=1000 + i)
            g2 = q.pack_gates(c2)
            s.reset()
            s.apply_circuit(g2)
            s.probabilities()
            cb += gate_bytes(c2)
        t_cold = time.perf_counter() - t0
        barrier()
        if dist:
            tt = torch.tensor([t_cold], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_cold = tt.item()
        e2e["cold"] = {"value": cb / t_cold / 1e9, "unit": UNIT, "steps": cold_steps,
                       "ms_per_step": t_cold / cold_steps * 1e3,
                       "ratio_to_warm": (t_cold / cold_steps) / (t_e2e / e2e_steps),
                       "what": "as e2e, but each step a circuit of the same recipe with a fresh seed (seeds 1000+i)"}

    # ---- roofline of the dominant kernel ----
    # Each launch has algorithmic bytes (HBM) and algorithmic fp64 flops; the
    # binding roofline is the one with the larger ideal time.  HBM peak:
    # MEASURED_PEAKS.json; fp64 peak: derived from unit counts and clock
    # (DESIGN.md "Rooflines"): 148 SMs x 64 FP64 FMA/clk x 2 flop x 1.965 GHz.
    peak, peak_src = peaks()
    peak_fp64 = ALU_PEAK_TFLOPS
    dom = max(prof.items(), key=lambda kv: kv[1]["ms"]) if prof else None
    roof = None
    per_kernel = {}
    for k, v in prof.items():
        per_kernel[k] = {"launches": v["launches"], "ms_total": v["ms"],
                         "avg_ms": v["ms"] / max(v["launches"], 1),
                         "GBps": v["bytes"] / max(v["ms"], 1e-9) / 1e6,
                         "TFLOPs": v["flops"] / max(v["ms"], 1e-9) / 1e9,
                         "share_of_step": v["ms"] / ms}
    if dom:
        k, v = dom
        sec = v["ms"] / 1e3
        gbs = v["bytes"] / sec / 1e9
        tfl = v["flops"] / sec / 1e12
        t_hbm = v["bytes"] / (peak * 1e9)
        t_alu = v["flops"] / (peak_fp64 * 1e12)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                t = json.load(open(tp)).get(k)
                traffic = t["dram_over_algorithmic"] * v["bytes"] / v["launches"] if t else None
            except Exception:
                traffic = None
        common = {"kernel": k, "traffic": traffic, "bytes_per_launch": v["bytes"] / v["launches"],
                  "flops_per_launch": v["flops"] / v["launches"], "avg_launch_ms": v["ms"] / v["launches"],
                  "hbm": {"achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak, "peak_source": peak_src},
                  "fp64": {"achieved": tfl, "peak": peak_fp64, "unit": "TFLOP/s", "frac": tfl / peak_fp64,
                           "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (measured DFMA "
                                          "microbenchmark: 33.6 TFLOP/s)"}}
        if t_alu > t_hbm:
            roof = {"bound": "alu", "achieved": tfl, "peak": peak_fp64, "unit": "TFLOP/s", "frac": tfl / peak_fp64,
                    **common}
        else:
            roof = {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak, **common}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_sample(circ)
        except Exception as ex:  # never let the baseline kill the bench line
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": name, "n_qubits": n, "gates_per_step": len(circ),
                           "amplitudes_per_gpu": 1 << (n - int(round(math.log2(world)))),
                           "fuse": args.fuse, "l2": "inputs larger than L2 (128 GiB state per GPU), no flush",
                           "parallelism": f"state sharded over {world} GPU(s) by the top log2(P) qubits; {mode}"},
                "gates_per_s": gates_per_s, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "exchange": exchange, "gpu_launches": launches, "clocks": clk, "per_kernel": per_kernel,
                "library": {"passes": st["passes"], "jit_passes": st["jit_passes"], "fused_gates": st["fused_gates"],
                            "sweeps": st["sweeps"],
                            "exchanges": st["exchanges"], "exchange_GB": st["exchange_bytes"] / 1e9}}
        emit(line)
    s.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
