#!/usr/bin/env python3
"""Benchmark of the qTask hot path on B200: full simulation of BASELINE.json
config 3 (30 qubits, 20 layers of U3 on every qubit + CZ brick-wall, 890
gates, 16 GiB complex128 state) -- the headline HBM-roofline config.

One step = |0...0> -> apply all 890 gates (seeded synthetic circuit; the
reference's QASMBench inputs are not available). Metric: amplitude-gate
updates/s = G * 2^n / t, whole job. The state (16 GiB) is larger than L2, so
no flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N   (sharded state, NCCL)

Keys beyond the driver contract: roofline (HBM, dominant kernel = the fused
tile pass), roofline_fp64, cpu_baseline, e2e, clocks, gpu_launches.
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

METRIC = "amplitude-gate updates/s"
UNIT = "amp-gate/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in self.rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in self.rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[5 + i].lower() == "active"})
        pw = [num(r[3]) for r in self.rows if num(r[3]) is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


def workload(name):
    from paper_2210_01076_b200 import workloads as W
    return {"c1": W.config1, "c2": W.config2, "c3": W.config3, "c4": W.config4,
            "c5": W.config5}[name]()


def cpu_reference(w, budget_s: float = 20.0):
    """The reference's own CPU implementation of the path on this host: the
    dense oracle (qtask::oracle::apply_gate_dense, oracle.cpp:15-50; single
    threaded by design), compiled from the reference sources
    (oracle/_ref), on a bounded prefix of the workload's logical gates."""
    import numpy as np

    import oracle
    from paper_2210_01076_b200.gates import lower_to_reference
    if not oracle.ref_available():
        return None
    # grow the sample until it costs ~budget_s (the first logical gates)
    count = 1
    secs = 0.0
    while True:
        sample = w.gates[:count]
        secs = oracle.ref_time_gates(w.n, lower_to_reference(sample), basis=w.basis)
        if secs >= budget_s / 3 or count >= len(w.gates):
            break
        count = min(len(w.gates), max(count + 1, int(count * budget_s / 3 / max(secs, 1e-3))))
    value = count * float(1 << w.n) / secs
    return {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"first {count} logical gates of {w.name} ({len(lower_to_reference(sample))} "
                      f"reference gates) on the 2^{w.n} state, reference oracle "
                      f"(oracle.cpp:15-50, single-threaded as written), {secs:.2f} s"}


def cpu_port_multicore(w, budget_s: float = 10.0):
    """The multithreaded restatement of the same dense kernel (oracle/qt_oracle.c,
    memcmp-identical to oracle.cpp:15-50; threads split the pair loop) on the
    first gates of the workload, all host threads: the honest multi-core CPU
    figure beside the reference's single-threaded one."""
    import numpy as np

    import oracle
    from paper_2210_01076_b200.gates import lower_to_reference
    threads = os.cpu_count() or 1
    st = np.zeros(1 << w.n, dtype=np.complex128)
    st[w.basis] = 1.0
    done = 0
    secs = 0.0
    count = 1
    while done < len(w.gates):
        sample = w.gates[done:done + count]
        t0 = time.perf_counter()
        oracle.simulate(w.n, lower_to_reference(sample), state=st, threads=threads)
        dt = time.perf_counter() - t0
        secs += dt
        done += len(sample)
        if secs >= budget_s:
            break
        count = max(1, int(count * min(4.0, (budget_s - secs) / max(dt, 1e-3) / 2)))
    return {"value": done * float(1 << w.n) / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {done} logical gates of {w.name} on the 2^{w.n} state, multithreaded "
                      f"oracle restatement (oracle/qt_oracle.c), {threads} threads, {secs:.2f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = workload(args.workload)
    vals = []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_reference(w, budget_s=min(20.0, 60.0 / max(1, args.steps + args.warmup)))
        if cb is None:
            print(json.dumps({"impl": "reference", "unavailable":
                              "oracle/_ref/libqtask_ref.so not built"}))
            return 0
        if i >= args.warmup:
            vals.append(cb["value"])
    value = statistics.median(vals)
    G = w.metric_gates
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": G * float(1 << w.n) / value * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic",
            "config": {"workload": w.name, "qubits": w.n, "gates": G,
                       "note": w.note},
            "cpu_baseline": dict(cb, value=value),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def latency_stats(xs):
    if not xs:
        return None
    s = sorted(xs)
    return {"mean_ms": statistics.mean(s), "median_ms": statistics.median(s),
            "p90_ms": s[min(len(s) - 1, int(0.9 * len(s)))], "count": len(s)}


def measure_incremental(make_sim, w, nmods, reference=False, tail_split=True):
    """Per-modifier latency through the Simulator API: host
    wall time from the start of the modifier calls to the return of
    update_state (device synchronised, numeric flag checked). Position class:
    config 5 alternates uniform / last-10% positions every two modifiers."""
    from paper_2210_01076_b200 import workloads as W
    sim = make_sim(w.n)
    drv = W.NetDriver(sim, reference_gates=reference)
    t0 = time.perf_counter()
    drv.build(w.gates)
    build_ms = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    sim.update_state()
    full_ms = (time.perf_counter() - t0) * 1e3
    # the GPU engine compiles the passes of its segments in the background
    # (hybrid compiled passes): the modifiers are timed on the warm engine
    bg_s = 0.0
    if not reference:
        from paper_2210_01076_b200 import jit_wait
        t0 = time.perf_counter()
        jit_wait(300)
        bg_s = time.perf_counter() - t0
    lat = {"uniform": [], "tail": []}
    for m, mod in enumerate(w.modifiers[:nmods]):
        cls = "tail" if (tail_split and (m // 2) % 2 == 1) else "uniform"
        t0 = time.perf_counter()
        drv.modify(mod)
        sim.update_state()
        lat[cls].append((time.perf_counter() - t0) * 1e3)
    nrm = sim.norm_squared()
    close = getattr(sim, "close", None)
    if close:
        close()
    out = {"build_ms": build_ms, "full_update_ms": full_ms,
           "uniform": latency_stats(lat["uniform"]), "tail": latency_stats(lat["tail"]),
           "norm_error": abs(nrm - 1.0)}
    if not reference:
        out["background_compile_wait_s"] = bg_s
    return out


def incremental_section(nmods_c5, nmods_c5_ref=4):
    """Config 5 (28 qubits, 5000 gates, alternating insert/remove) on the GPU
    engine, with its CPU references: the reference engine on the same
    generator at reduced n (and the GPU engine beside it) and the
    multithreaded oracle's full re-simulation at 28 qubits; config 1 (16
    qubits, 400 gates + 20 modifiers) on the GPU engine and on the reference
    engine (qtask::Simulator, all host threads)."""
    import oracle
    from paper_2210_01076_b200 import Config, Simulator
    from paper_2210_01076_b200 import workloads as W
    out = {}
    w5 = W.config5()
    out["c5_gpu"] = dict(measure_incremental(lambda n: Simulator(n, Config()), w5, nmods_c5),
                         workload=w5.name, modifiers=nmods_c5)
    w1 = W.config1()
    out["c1_gpu"] = dict(measure_incremental(lambda n: Simulator(n, Config()), w1, 20,
                                             tail_split=False), workload=w1.name)
    threads = os.cpu_count() or 1
    if oracle.ref_available():
        # C5's generator at the largest n the reference engine holds in a
        # bounded run (n = 16: 2^8 blocks of 256; its memory is O(stages x
        # 2^n), 7 GiB here, and n = 28 is out of reach), beside the GPU
        # engine on the identical reduced-n workload
        w5r = W.config5(n=16, nmods=max(4, nmods_c5_ref))
        out["c5_reference_cpu_reduced_n"] = dict(
            measure_incremental(lambda n: oracle.RefSimulator(n, 256, 0), w5r, nmods_c5_ref,
                                reference=True),
            workload=w5r.name + "@n=16", cores=threads, block_size=256, modifiers=nmods_c5_ref,
            note="REDUCED n (16 instead of 28): the reference qtask::Simulator (engine.cpp, "
                 "compiled from its sources) on C5's generator -- 5000 gates, alternating "
                 "insert / remove, uniform / last-10% positions -- threads = "
                 "hardware_concurrency; CZ as H,CX,H nets")
        out["c5_gpu_reduced_n"] = dict(
            measure_incremental(lambda n: Simulator(n, Config()), w5r, nmods_c5_ref),
            workload=w5r.name + "@n=16", modifiers=nmods_c5_ref,
            note="the GPU engine on the identical reduced-n workload")
    # the non-incremental CPU figure at the real size: the multithreaded
    # restated oracle (bit-identical to the reference's oracle.cpp) re-simulating
    # C5 at 28 qubits, timed on a prefix and scaled to the 5000 gates
    # (oracle time is linear in the gate count)
    import numpy as np
    sample = 40
    st = np.zeros(1 << w5.n, dtype=np.complex128)
    st[0] = 1.0
    from paper_2210_01076_b200.gates import lower_to_reference
    ref_gates = lower_to_reference(w5.gates)
    t0 = time.perf_counter()
    oracle.simulate(w5.n, ref_gates[:sample], state=st, threads=threads)
    per_gate = (time.perf_counter() - t0) / sample
    del st
    out["c5_oracle_cpu_n28"] = {
        "full_resimulation_ms": per_gate * len(ref_gates) * 1e3,
        "per_reference_gate_ms": per_gate * 1e3, "sample_gates": sample,
        "reference_gates": len(ref_gates), "cores": threads,
        "note": "NON-INCREMENTAL CPU: the multithreaded oracle restatement (oracle/qt_oracle.c, "
                "memcmp-identical to oracle.cpp:15-50) re-simulating C5 at 28 qubits from "
                "|0...0>, timed on the first 40 reference gates and scaled to all; a full run "
                "measured 350 s at 16 threads (profiles/r02_c5_full_size.json)"}
    if oracle.ref_available():
        out["c1_reference_cpu"] = dict(
            measure_incremental(lambda n: oracle.RefSimulator(n, 256, 0), w1, 20,
                                reference=True, tail_split=False),
            workload=w1.name, cores=threads, block_size=256,
            note="reference qtask::Simulator (engine.cpp) compiled from its sources, "
                 "threads = hardware_concurrency; CZ as H,CX,H nets")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--tile-qubits", type=int, default=0)
    ap.add_argument("--mode", default="compiled", choices=["compiled", "interpreted"],
                    help="compiled: every tile pass is an NVRTC-compiled straight-line kernel "
                         "(built during warm-up, cached by source); interpreted: the lean "
                         "kernel interprets layer words")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hbm-bound", action="store_true",
                    help="skip the HBM-bound context measurement (config 5 as one full simulation)")
    ap.add_argument("--incremental-mods", type=int, default=24,
                    help="config-5 modifiers measured after the headline (0: skip)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    from paper_2210_01076_b200 import StateVector, jit_stats, nccl_unique_id, probe_fp64
    compiled = args.mode == "compiled"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        st = StateVector(workload(args.workload).n, mode="sharded", rank=rank, world=world,
                         nccl_id=bytes(idt.cpu().numpy().tobytes()), device=local,
                         tile_qubits=args.tile_qubits, compiled=compiled)
    else:
        dist = None
        st = StateVector(workload(args.workload).n, device=local, tile_qubits=args.tile_qubits,
                         compiled=compiled)
    w = workload(args.workload)
    n, G = w.n, w.metric_gates
    amps = float(1 << n)

    stream = torch.cuda.ExternalStream(st.stream_ptr, device=torch.device("cuda", local))

    def step():
        st.set_basis(w.basis)
        st.apply(w.gates)

    # warm-up: the first step plans on the host (compiled mode: a parallel
    # search over the planner's per-pass FP64 cap) and compiles each pass
    # (NVRTC, parallel) into the process cache; later steps apply the same
    # gate list from the same qubit map, so the state's 1-entry plan cache
    # returns the previous plan, lowering and kernels (no host planning)
    j0 = jit_stats()
    tw = time.perf_counter()
    step()
    st.sync()
    first_step_ms = (time.perf_counter() - tw) * 1e3
    for _ in range(args.warmup - 1):
        step()
    st.sync()
    j1 = jit_stats()
    plan = json.loads(st.plan_json(w.gates))
    tiles = [p for p in plan["passes"] if p["kind"] == "tile"]

    # ---- timed region: K steps, CUDA events on the library's stream --------
    st.set_timing(True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    pass_ms = []
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    # per-launch events recorded on the same stream inside the timed region
    timings = st.last_timings()
    pass_ms = [ms for kind, ms in timings if kind == 0]
    exch_ms = [ms for kind, ms in timings if kind == 1]
    run_stats = st.stats()
    st.sync()
    ms = e0.elapsed_time(e1)
    st.set_timing(False)
    t = torch.tensor([ms, sum(exch_ms) / max(1, args.steps)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms = float(t[0].item())
    exch_ms_step = float(t[1].item())
    sec = ms / 1e3
    value = args.steps * G * amps / sec
    launches = args.steps * (len(tiles) + 1 + sum(len(p.get("swap", []))
                                                  for p in plan["passes"]
                                                  if p["kind"] == "exchange"))
    j2 = jit_stats()

    # ---- e2e through the public API: host gate list in, norm + amplitudes out
    head = 1 << 16
    buf = np.empty(head, dtype=np.complex128)
    e2e_steps = max(1, min(args.steps, 3))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        st.set_basis(w.basis)
        st.apply(w.gates)                  # gate array copied from host memory
        nrm = st.norm_squared()            # D2H of the reduction
        st.read(0, head, buf)              # D2H of 2^16 amplitudes
    e2e_sec = time.perf_counter() - t0
    tt = torch.tensor([e2e_sec], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_sec = float(tt.item())

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    hbm_peak, peak_kind = load_peaks()
    traffic = None  # DRAM bytes per launch of the dominant kernel, from an ncu --set full capture
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        if ("qtjit" in tj.get("kernel", "")) == compiled and args.workload == "c3" and world == 1:
            traffic = float(tj["bytes_per_launch"])
    except (OSError, ValueError, KeyError):
        pass
    avg_pass_ms = statistics.mean(pass_ms) if pass_ms else float("nan")
    local_amps = amps / world
    bytes_per_pass = 32.0 * local_amps
    achieved_gbs = bytes_per_pass / (avg_pass_ms * 1e-3) / 1e9
    fp64_ops = sum(p["fp64_per_amp"] for p in tiles) * local_amps
    pass_total_ms = sum(pass_ms) / max(1, args.steps)
    try:
        fp64_peak = probe_fp64(local)  # DFMA-pipe instructions / s
    except Exception:
        fp64_peak = float("nan")
    fp64_achieved = fp64_ops / (pass_total_ms * 1e-3)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic",
        "config": {"workload": w.name, "qubits": n, "gates": G,
                   "state_bytes": int(16 * amps), "l2": "inputs larger than L2 (16 GiB state)",
                   "parallelism": f"sharded{world}" if world > 1 else "single",
                   "passes_per_step": len(tiles), "note": w.note},
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak,
                     "unit": "GB/s", "frac": achieved_gbs / hbm_peak, "traffic": traffic,
                     "kernel": ("qtjit: compiled tile passes (qt_jit.cpp)" if compiled
                                else "tile_pass_kernel (qt_tilepass.cu)"), "peak_kind": peak_kind,
                     "bytes_per_launch": bytes_per_pass, "avg_launch_ms": avg_pass_ms,
                     "note": "the time-optimal plan packs the gates into few FP64-bound passes (%d FP64 "
                             "ops per amplitude over %d passes), so the HBM fraction per pass is low "
                             "by construction: see roofline_fp64, profiles/r02_ablation.md (the ring "
                             "streams at 0.90 of this peak without arithmetic) and DESIGN.md section 4"
                             % (round(sum(p["fp64_per_amp"] for p in tiles)), len(tiles))},
        "roofline_fp64": {"achieved_dfma_per_s": fp64_achieved, "peak_dfma_per_s": fp64_peak,
                          "frac": fp64_achieved / fp64_peak if fp64_peak else None,
                          "note": "DFMA-pipe instructions of the lowered ops (complex 2x2 = 8/amp, "
                                  "real rotation = 2/amp in scaled form, diagonal table of unit "
                                  "phases = 3/amp as shears, complex table = 4/amp); peak from an "
                                  "FMA-chain probe on this GPU (16 chains per thread, 64 warps "
                                  "per SM)"},
        "mode": args.mode,
        "compile": {"passes_compiled": j1["compiled"] - j0["compiled"],
                    "compile_ms": j1["compile_ms"] - j0["compile_ms"],
                    "first_step_ms": first_step_ms,
                    "timed_region_compiles": j2["compiled"] - j1["compiled"],
                    "timed_region_cache_hits": j2["cache_hits"] - j1["cache_hits"],
                    "note": "compiled mode: the plan search and the NVRTC compile of every "
                            "pass happen in the first warm-up step (outside the timed region); "
                            "timed steps re-apply the same gate list from the same qubit map "
                            "and reuse that plan, its lowering and kernels through the state's "
                            "1-entry plan cache (no host planning, no cache lookups)"},
        "e2e": {"value": e2e_steps * G * amps / e2e_sec, "unit": UNIT,
                "h2d_bytes_per_step": int(w.gates.nbytes),
                "d2h_bytes_per_step": int(8 + 16 * head),
                "note": "set_basis + apply (host gate array, plan reused) + norm + 2^16 "
                        "amplitudes read back, host wall clock per step"},
        "e2e_cold": {"value": G * amps / (first_step_ms * 1e-3), "unit": UNIT, "ms": first_step_ms,
                     "disk_cache_hits": j1.get("disk_hits", 0) - j0.get("disk_hits", 0),
                     "note": "the first apply of this process through the public API: lowering, "
                             "the plan search, code generation and the compile of every pass (NVRTC, "
                             "or the on-disk cubin cache when this box compiled the passes before), "
                             "then the passes; one-shot users without a warm cache pay this"},
        "check": {"norm_error": abs(nrm - 1.0),
                  "note": "|<psi|psi> - 1| of the last e2e step's state (deterministic "
                          "two-level reduction)"},
        "exchange": ({
            "swaps_per_step": int(run_stats["swaps"]),
            "sent_bytes_per_step_per_gpu": int(run_stats["exchanged_bytes"]),
            "local_copy_bytes_per_step_per_gpu": int(run_stats["exchange_local_bytes"]),
            "device_ms_per_step": exch_ms_step,
            "ms_per_swap": exch_ms_step / max(1, run_stats["swaps"]),
            "nvlink_gbs_per_gpu": (run_stats["exchanged_bytes"] / (exch_ms_step * 1e-3) / 1e9
                                   if exch_ms_step > 0 else None),
            "nvlink_frac": (run_stats["exchanged_bytes"] / (exch_ms_step * 1e-3) / 900e9
                            if exch_ms_step > 0 else None),
            "nvlink_peak_note": "900 GB/s per direction per GPU (nominal NVLink 5); the "
                                "measured peer copy on this pool is ~770 GB/s",
            "transport": "NCCL grouped send/recv, two-buffer exchange (received regions land "
                         "in place; only this rank's own region is copied locally)",
        } if world > 1 else None),
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if compiled and world == 1:
        # the same steps through the interpreter kernel, for comparison
        st.close()
        sti = StateVector(n, device=local, tile_qubits=args.tile_qubits, compiled=False)
        si = torch.cuda.ExternalStream(sti.stream_ptr, device=torch.device("cuda", local))
        for _ in range(2):
            sti.set_basis(w.basis)
            sti.apply(w.gates)
        sti.sync()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(si)
        for _ in range(args.steps):
            sti.set_basis(w.basis)
            sti.apply(w.gates)
        f1.record(si)
        torch.cuda.synchronize()
        ims = f0.elapsed_time(f1) / args.steps
        sti.close()
        line["interpreted"] = {"ms_per_step": ims, "value": G * amps / (ims * 1e-3),
                               "kernel": "tile_pass_kernel (qt_tilepass.cu, layer-word interpreter)"}
    if compiled and world == 1 and args.workload == "c3" and not args.no_hbm_bound:
        # the HBM-bound workload class beside the FP64-bound headline: BASELINE
        # config 5's circuit (28 q, 5000 random gates) as one full simulation;
        # its passes are light, so their time is the streaming time plus what
        # the kernel fails to hide
        try:
            w5 = workload("c5")
            s5 = StateVector(w5.n, device=local, compiled=True)
            s5.set_timing(True)
            for _ in range(2):
                s5.set_basis(w5.basis)
                s5.apply(w5.gates)
                s5.sync()
                t5 = [ms for kind, ms in s5.last_timings() if kind == 0]
            s5.close()
            avg5 = statistics.mean(t5)
            gbs5 = 32.0 * float(1 << w5.n) / (avg5 * 1e-3) / 1e9
            line["roofline_hbm_bound"] = {
                "workload": w5.name, "qubits": w5.n, "passes": len(t5), "ms_per_step": sum(t5),
                "avg_launch_ms": avg5, "achieved": gbs5, "peak": hbm_peak, "unit": "GB/s",
                "frac": gbs5 / hbm_peak,
                "note": "same ring kernel on a random circuit (about 66 gates per pass): the passes "
                        "are HBM-bound; second apply, CUDA events per pass"}
        except Exception as e:  # context only, never fatal for the headline line
            line["roofline_hbm_bound"] = {"error": f"{type(e).__name__}: {e}"}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference(w)
        line["cpu_multicore"] = cpu_port_multicore(w)
    if world == 1 and args.incremental_mods > 0:
        st.close()  # free the 16 GiB state for the incremental engine's checkpoints
        try:
            line["incremental"] = incremental_section(args.incremental_mods)
        except Exception as e:  # reported, never fatal for the headline line
            line["incremental"] = {"error": f"{type(e).__name__}: {e}"}
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
