#!/usr/bin/env python3
"""Benchmark of the per-window Network Sensing Graph Challenge path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C2|C3|C1]

One step = one pass of the whole hot path (partition -> link buckets -> side buckets -> the nine
statistics of every window) over one batch of windows:
  N = 1 (default workload C2): one C2 batch, 64 windows x 2^17 packets, Zipf(s=1.1, K=2^20) IPv4 pairs
        from the seeded counter-based generator, generated on the device; steps cycle through a 1 GiB ring
        of 16 such batches, so every step reads inputs that are not L2-resident (126 MB L2).
  N > 1 (default workload C4, torchrun, one rank per GPU, NCCL): the 2^30-packet C4 input (8192
        windows) split into contiguous window blocks, one per rank, resident in HBM; one call per rank
        per step over its whole block, then the NCCL all_gather_into_tensor of the 72 B/window result rows
        inside the timed region (strong scaling; the line also reports the rate without the gather).

The JSON line carries: value (device-timed aggregate packets/s, max over ranks), e2e (the same
metric through the public API from pinned HOST buffers, H2D + D2H inside the timed region),
roofline (HBM: 8 B/packet + 72 B/window algorithmic bytes over the persistent kernel's CUDA-event
time), cpu_baseline (the CPU oracle on a bounded sample, rank 0 at N=1), clocks and gpu_launches.
`--impl reference` times the CPU oracle itself (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "packets/sec (device-timed, max over ranks) at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "packets/s"
WINDOW = 1 << 17
WINDOWS_PER_STEP = 64
RING = 16
BYTES_PER_PACKET = 8          # algorithmic: one packed u64 key (src<<32|dst) read once
BYTES_PER_WINDOW_OUT = 72     # nine u64 per window written
C4_PACKETS = 1 << 30          # BASELINE configs[3]: 8192 windows


def workload(name: str):
    import gen

    if name == "C2":
        return gen.Dist("zipf", 1.1, 1 << 20), 2, "C2: Zipf(s=1.1, K=2^20) IPv4 pairs, seed 2"
    if name == "C4":
        return gen.Dist("zipf", 1.1, 1 << 20), 4, "C4: 2^30 packets (8192 windows), Zipf(s=1.1, K=2^20), seed 4"
    if name == "C3":
        return gen.Dist("heavy"), 3, "C3: heavy skew (Bernoulli(1/2) source 10.0.0.1, uniform dst), seed 3"
    if name == "C1":
        return gen.Dist("uniform"), 1, "C1-shaped: uniform 32-bit src/dst, seed 1"
    if name in ("Z08", "Z13", "Z15"):  # SURVEY §8(d) optional sweep of the Zipf exponent
        z = {"Z08": 0.8, "Z13": 1.3, "Z15": 1.5}[name]
        return gen.Dist("zipf", z, 1 << 20), 2, f"{name}: Zipf(s={z}, K=2^20) IPv4 pairs, seed 2"
    raise SystemExit(f"unknown workload {name}")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy, burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_per_launch(workload_name: str):
    """dram__bytes_read+write per call (all kernels of one call) from the committed ncu capture
    profiles/ncu_traffic.json, only if it was taken on the build being benched (same build id)."""
    from paper_2509_03653_b200 import _lib

    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
    except Exception:
        return None, "no profiles/ncu_traffic.json"
    e = t.get(workload_name)
    if e is None:
        return None, f"no entry for {workload_name}"
    if e.get("build_id") != _lib.build_id():
        return None, f"stale: captured on build {e.get('build_id')}, benching {_lib.build_id()}"
    return float(e["dram_bytes_per_call"]), f"ncu capture of build {e['build_id']} ({e.get('source', '')})"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(dist, seed, budget_s: float = 10.0):
    """The CPU oracle (O2) on a bounded sample of the same workload: all host threads, and one thread."""
    import gen
    import oracle

    threads = oracle.hardware_threads()
    done_pkts, t_total, w = 0, 0.0, 0
    batch = WINDOWS_PER_STEP
    while t_total < budget_s and w < 128 * batch:
        keys = gen.generate_host(dist, seed, w * WINDOW, batch * WINDOW, packed=True)
        t0 = time.perf_counter()
        oracle.window_stats_sort(keys=keys, window=WINDOW, threads=threads)
        t_total += time.perf_counter() - t0
        done_pkts += batch * WINDOW
        w += batch
    one = gen.generate_host(dist, seed, 0, 8 * WINDOW, packed=True)
    t0 = time.perf_counter()
    oracle.window_stats_sort(keys=one, window=WINDOW, threads=1)
    t1 = time.perf_counter() - t0
    return {"value": done_pkts / t_total, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{w} windows x 2^17 packets of the same stream (O2 std::sort oracle, {threads} threads, "
                      f"{t_total:.1f} s)",
            "value_1core": 8 * WINDOW / t1, "sample_1core": f"8 windows x 2^17 packets, 1 thread, {t1:.2f} s",
            "cpu_model": cpu_model()}


def spot_check(dist, seed, got_rows, first_packet: int, windows):
    """After the timed region: windows of the last step's device output against the oracle on the same
    windows regenerated on the host (gen's host generator, which the device generator is pinned to)."""
    import numpy as np

    import gen
    import oracle

    ok = True
    for w in windows:
        keys = gen.generate_host(dist, seed, first_packet + w * WINDOW, WINDOW, packed=True)
        want = oracle.window_stats_sort(keys=keys, window=WINDOW)[0]
        ok = ok and np.array_equal(got_rows[w].view(np.uint64), want)
    return {"windows": [int(w) for w in windows], "match": bool(ok), "oracle": "O2 (std::sort)"}


def run_reference(args):
    """Reference arm of this tier: the CPU oracle as it stands, timed on the host cores."""
    import gen
    import oracle

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    dist_, seed, desc = workload(args.workload)
    threads = oracle.hardware_threads()
    # windows per reference step: a C2 batch (64 windows), and at least one window per host thread
    per_step = max(WINDOWS_PER_STEP, threads)
    samples = [gen.generate_host(dist_, seed, i * per_step * WINDOW, per_step * WINDOW, packed=True)
               for i in range(min(4, args.steps + args.warmup))]
    for i in range(args.warmup):
        oracle.window_stats_sort(keys=samples[i % len(samples)], window=WINDOW, threads=threads)
    t0 = time.perf_counter()
    for i in range(args.steps):
        oracle.window_stats_sort(keys=samples[i % len(samples)], window=WINDOW, threads=threads)
    dt = time.perf_counter() - t0
    pkts = args.steps * per_step * WINDOW
    value = pkts / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": desc + f" ({per_step} windows of 2^17 packets per step: bounded CPU sample)",
                   "window": WINDOW},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{per_step} windows per step x {args.steps} steps, O2 oracle, {threads} threads",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default=None, help="C2 (default at N=1), C4 (default at N>1), C3, C1, Z08/13/15")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--once", action="store_true", help="a single untimed call (for ncu)")
    ap.add_argument("--path", choices=["windows", "trace", "anonymize"], default="windows",
                    help="windows: per-window statistics (north_star); trace: the whole-trace statistics of each "
                         "step's packets (nsg_trace_stats; N>1: distributed_trace_stats with all-to-all exchanges, "
                         "SURVEY §8(f) f4b); anonymize: relabel every address of each step's packets "
                         "(nsg_anonymize, one shuffle round, SURVEY §8(f) f2)")
    ap.add_argument("--l2", choices=["cold", "warm"], default="cold",
                    help="cold: steps cycle through a 1 GiB ring of batches (never L2-resident; the default and the "
                         "headline); warm: one 64 MiB batch reused every step (L2-resident input, SURVEY §8(d))")
    ap.add_argument("--streams", type=int, default=3,
                    help="default path at N=1: consecutive batches alternate over this many CUDA streams with "
                         "their own workspaces, so a batch's pipeline fill overlaps the previous batch's drain")
    ap.add_argument("--graphs", type=int, default=1,
                    help="default path at N=1: each call of the hot path is captured once in a CUDA graph (one per "
                         "ring batch and stream) and replayed every step (same kernels and work, lower launch "
                         "overhead); 0 = plain calls")
    ap.add_argument("--transport", choices=["nccl", "p2p"], default="nccl",
                    help="N>1: NCCL collectives, or the kernels storing straight into the other ranks' "
                         "CUDA-IPC-mapped buffers over peer memory (windows: result rows from the epilogue; "
                         "trace: the partition / record emission)")
    ap.add_argument("--input", choices=["packets", "weighted"], default="packets",
                    help="packets: raw packets (north_star); weighted: rows (src, dst, n_packets) with n_packets "
                         "uniform in [1, 8] (nsg_window_stats_weighted, SURVEY §8(f) f4a); unit = rows/s")
    ap.add_argument("--outputs", choices=["stats", "vectors"], default="stats",
                    help="stats: the nine statistics (north_star); vectors: + per-window link / source / "
                         "destination vectors and IP set counts (nsg_window_vectors, SURVEY §8(f) f1, f3)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.workload is None:
        args.workload = "C2" if int(os.environ.get("WORLD_SIZE", "1")) == 1 else "C4"
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as tdist

    import gen
    import paper_2509_03653_b200 as nsg
    from paper_2509_03653_b200.distributed import gather_window_stats

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N>1 must be launched with torchrun (one rank per GPU)")
    local = local % max(1, torch.cuda.device_count())  # NSG_BENCH_BACKEND=gloo may share one GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("NSG_BENCH_BACKEND", "nccl")  # "gloo": test the N>1 path on one GPU
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=dev)
        else:
            tdist.init_process_group(backend)
    dist_, seed, desc = workload(args.workload)

    c4 = args.workload == "C4"
    if c4:  # the whole C4 input, this rank's contiguous window block resident in HBM (> L2 at any N <= 8)
        from paper_2509_03653_b200.distributed import packet_block

        c4_p0, c4_p1 = packet_block(C4_PACKETS, WINDOW, rank, world)
        n = c4_p1 - c4_p0
        wps, total_windows, ring_n = n // WINDOW, C4_PACKETS // WINDOW, 1
        ring = torch.empty((1, n), dtype=torch.int64, device=dev)
        gen.generate_device(dist_, seed, c4_p0, n, keys=ring[0])
        first_packet = lambda i: c4_p0  # noqa: E731
    else:
        n = WINDOWS_PER_STEP * WINDOW
        wps, total_windows = WINDOWS_PER_STEP, WINDOWS_PER_STEP * world
        # this rank's ring: batch i of rank r covers packets [((i * world) + r) * n, ...) of the stream
        ring_n = RING if args.l2 == "cold" else 1
        ring = torch.empty((ring_n, n), dtype=torch.int64, device=dev)
        for i in range(ring_n):
            gen.generate_device(dist_, seed, ((i * world) + rank) * n, n, keys=ring[i])
        first_packet = lambda i: (((i % ring_n) * world) + rank) * n  # noqa: E731
    torch.cuda.synchronize(dev)
    ws = nsg.Workspace(n, WINDOW, dev)
    outs = [torch.empty((wps, 9), dtype=torch.int64, device=dev) for _ in range(RING)]
    vec = args.outputs == "vectors"
    wtd = args.input == "weighted"
    p2p_tab = None
    if world > 1 and args.transport == "p2p":  # the result gather done by the kernels' epilogues (peer memory)
        from paper_2509_03653_b200.distributed import PeerBuffers

        p2p_tab = PeerBuffers(total_windows * 9, None, dev)
    trace = args.path == "trace"
    anon = args.path == "anonymize"
    if c4 and (trace or anon or vec or wtd or args.transport != "nccl"):
        raise SystemExit("--workload C4: the per-window statistics with the NCCL gather only")
    if anon and (vec or wtd or world > 1):
        raise SystemExit("--path anonymize: one GPU, --input packets --outputs stats only")
    if trace and (vec or wtd):
        raise SystemExit("--path trace supports --input packets --outputs stats only")
    from paper_2509_03653_b200.distributed import distributed_trace_stats
    if wtd and vec:
        raise SystemExit("--input weighted supports --outputs stats only")
    wring = None
    if wtd:  # n_packets per row, seeded, uniform in [1, 8]
        gw = torch.Generator(device=dev)
        gw.manual_seed(1000 + seed + rank)
        wring = torch.randint(1, 9, (ring_n, n), generator=gw, device=dev, dtype=torch.int32)
    vbuf = nsg.window_vectors(ring[0], WINDOW, out=outs[0], workspace=ws) if vec else None
    if args.once:
        if vec:
            nsg.window_vectors(ring[0], WINDOW, out=outs[0], workspace=ws, buffers=vbuf)
        else:
            nsg.window_stats_packed(ring[0], WINDOW, out=outs[0], workspace=ws)
        torch.cuda.synchronize(dev)
        return 0

    # Plain per-window statistics: batches alternate over `nstreams` streams (double-buffered workspaces);
    # each call is still one whole pass of the hot path over its batch.  At N>1 the result gathers stay on
    # one stream of their own, in step order (one communicator is never driven from two streams at once).
    nstreams = max(1, args.streams) if not (anon or trace or c4) and (world == 1 or not (vec or wtd)) else 1
    wss = [ws] + [nsg.Workspace(n, WINDOW, dev) for _ in range(nstreams - 1)]
    vbufs = [vbuf] + ([nsg.window_vectors(ring[0], WINDOW, out=outs[1], workspace=wss[1]) for _ in range(nstreams - 1)]
                      if vec else [None] * (nstreams - 1))
    use_graphs = bool(args.graphs) and world == 1 and not (vec or wtd or trace or anon or c4)
    # (graphs are captured on non-default streams)
    streams = ([] if use_graphs else [torch.cuda.current_stream(dev)])
    streams += [torch.cuda.Stream(dev) for _ in range(nstreams - len(streams))]
    cur_stream = torch.cuda.current_stream(dev)
    gstream = torch.cuda.Stream(dev) if (nstreams > 1 and world > 1) else None

    graphs = []
    last_out = [outs[0]]

    def step(i, evs=None):
        if use_graphs and graphs:  # the captured call of batch (i mod ring) on stream (i mod nstreams)
            j = i % len(graphs)
            s_i = streams[j % nstreams]
            with torch.cuda.stream(s_i):
                if evs:
                    evs[0].record()
                graphs[j].replay()
                if evs:
                    evs[1].record()
            last_out[0] = outs[j % RING]
            return outs[j % RING]
        last_out[0] = outs[i % RING]
        if nstreams > 1:
            s_i = streams[i % nstreams]
            with torch.cuda.stream(s_i):
                if vec or wtd:  # events around the whole call (workspace reset + persistent kernel + check)
                    if evs:
                        evs[0].record()
                    if vec:
                        r = nsg.window_vectors(ring[i % ring_n], WINDOW, out=outs[i % RING], workspace=wss[i % nstreams],
                                               buffers=vbufs[i % nstreams], stream=s_i)["stats"]
                    else:
                        r = nsg.window_stats_weighted(ring[i % ring_n], wring[i % ring_n], WINDOW, out=outs[i % RING],
                                                      workspace=wss[i % nstreams], stream=s_i)
                    if evs:
                        evs[1].record()
                    return r
                if world > 1 and args.transport == "p2p":
                    if evs:
                        evs[0].record()
                    r = nsg.window_stats_mirrored(ring[i % ring_n], p2p_tab.ptrs, rank * WINDOWS_PER_STEP, WINDOW,
                                                  out=outs[i % RING], workspace=wss[i % nstreams])
                    if evs:
                        evs[1].record()
                    return r
                r = nsg.window_stats_packed(ring[i % ring_n], WINDOW, out=outs[i % RING], workspace=wss[i % nstreams],
                                            stream=s_i, kernel_events=evs)
            if gstream is not None:
                gstream.wait_stream(s_i)
                with torch.cuda.stream(gstream):
                    gather_window_stats(r, total_windows)
            return r
        if anon:  # events around the whole call (bitmap reset + mark + rank prefix + relabel)
            if evs:
                evs[0].record()
            r = nsg.anonymize(ring[i % ring_n], seed=i, rounds=1)
            if evs:
                evs[1].record()
            return r
        if trace:  # events around the whole call (table resets + the trace kernels [+ exchanges])
            if evs:
                evs[0].record()
            r = nsg.trace_stats(ring[i % ring_n]) if world == 1 else \
                distributed_trace_stats(ring[i % ring_n], transport=args.transport)
            if evs:
                evs[1].record()
            return r
        if vec:  # events around the whole call (workspace reset + persistent kernel + overflow check)
            if evs:
                evs[0].record()
            r = nsg.window_vectors(ring[i % ring_n], WINDOW, out=outs[i % RING], workspace=ws, buffers=vbuf)["stats"]
            if evs:
                evs[1].record()
        elif wtd:  # events around the whole call (workspace reset + persistent kernel + overflow check)
            if evs:
                evs[0].record()
            r = nsg.window_stats_weighted(ring[i % ring_n], wring[i % ring_n], WINDOW, out=outs[i % RING], workspace=ws)
            if evs:
                evs[1].record()
        elif world > 1 and args.transport == "p2p":  # rows stored into every rank's IPC-mapped table
            if evs:  # events around the whole call (workspace reset + persistent kernel + overflow check)
                evs[0].record()
            r = nsg.window_stats_mirrored(ring[i % ring_n], p2p_tab.ptrs, rank * WINDOWS_PER_STEP, WINDOW,
                                          out=outs[i % RING], workspace=ws)
            if evs:
                evs[1].record()
            return r
        else:
            r = nsg.window_stats_packed(ring[i % ring_n], WINDOW, out=outs[i % RING], workspace=ws, kernel_events=evs)
        if world > 1:
            gather_window_stats(r, total_windows)
        return r

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)
    launches = nsg.last_launches()
    diag = ws.diag()
    if use_graphs:  # capture one call per (ring batch, stream) pair, after the warm-up initialised the library
        import math

        for j, s_j in enumerate(streams):  # the library's per-stream state exists before capture
            with torch.cuda.stream(s_j):
                nsg.window_stats_packed(ring[j % ring_n], WINDOW, out=outs[j % RING], workspace=wss[j], stream=s_j)
        torch.cuda.synchronize(dev)
        for j in range(ring_n * nstreams // math.gcd(ring_n, nstreams)):
            s_j = streams[j % nstreams]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s_j):
                nsg.window_stats_packed(ring[j % ring_n], WINDOW, out=outs[j % RING], workspace=wss[j % nstreams],
                                        stream=s_j)
            graphs.append(g)
        launches = nsg.last_launches()
        for i in range(len(graphs)):  # warm replays
            step(i)
        torch.cuda.synchronize(dev)

    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize(dev)
    wall0 = time.perf_counter()
    start.record()
    for s_ in streams:
        if s_ != cur_stream:
            s_.wait_event(start)
    for i in range(args.steps):
        step(i, kev[i])
    for s_ in streams + ([gstream] if gstream is not None else []):
        if s_ != cur_stream:
            cur_stream.wait_stream(s_)
    if p2p_tab is not None:  # every rank's rows are in every table before the clock stops
        torch.cuda.synchronize(dev)
        tdist.barrier()
    end.record()
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - wall0
    if world > 1:
        tdist.barrier()
    clocks = sampler.stop() if sampler else None
    t_ms = start.elapsed_time(end)
    k_ms = [a.elapsed_time(b) for a, b in kev]
    k_avg = sum(k_ms) / len(k_ms)
    coll_dev = dev if world > 1 and tdist.get_backend() == "nccl" else torch.device("cpu")
    if world > 1:
        tt = torch.tensor([t_ms, k_avg], dtype=torch.float64, device=coll_dev)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        t_ms, k_avg = float(tt[0]), float(tt[1])
    pkts_per_step = C4_PACKETS if c4 else n * world
    total_pkts = pkts_per_step * args.steps
    value = total_pkts / (t_ms / 1e3)
    value_no_gather = pkts_per_step / (k_avg / 1e3)  # kernels only (per-step CUDA events, max over ranks)
    last_rows = last_out[0].cpu().numpy()

    # ---- e2e: the public API from pinned host buffers (H2D of the keys + D2H of the result inside)
    host = ring[0].cpu().pin_memory()
    keys_dev = torch.empty(n, dtype=torch.int64, device=dev)
    out_host = torch.empty((wps, 9), dtype=torch.int64, pin_memory=True)
    e2e_steps = 3 if c4 else max(3, min(args.steps, 50))
    if vec:  # H2D of the keys, the call, D2H of the statistics and every vector array
        vhost = {k: torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for k, t in vbuf.items() if k != "stats"}

        def e2e_once():
            keys_dev.copy_(host, non_blocking=True)
            r = nsg.window_vectors(keys_dev, WINDOW, out=outs[0], workspace=ws, buffers=vbuf)
            out_host.copy_(r["stats"], non_blocking=True)
            for k, t in vhost.items():
                t.copy_(r[k], non_blocking=True)
        d2h_bytes = WINDOWS_PER_STEP * 9 * 8 + sum(t.numel() * t.element_size() for t in vhost.values())
    elif anon:  # H2D of the packets, the call, D2H of the relabelled src/dst and N
        ahost = torch.empty((2, n), dtype=torch.int32, pin_memory=True)

        def e2e_once():
            keys_dev.copy_(host, non_blocking=True)
            a, b, _ = nsg.anonymize(keys_dev, seed=1, rounds=1)
            ahost[0].copy_(a, non_blocking=True)
            ahost[1].copy_(b, non_blocking=True)
        d2h_bytes = 8 * n + 8
    elif trace:  # H2D of the packets, the whole-trace call, D2H of the nine statistics
        tout_host = torch.empty(9, dtype=torch.int64, pin_memory=True)

        def e2e_once():
            keys_dev.copy_(host, non_blocking=True)
            r = nsg.trace_stats(keys_dev) if world == 1 else distributed_trace_stats(keys_dev, transport=args.transport)
            tout_host.copy_(r, non_blocking=True)
        d2h_bytes = 9 * 8
    elif wtd:  # H2D of the rows (keys + n_packets), the call, D2H of the statistics
        whost = wring[0].cpu().pin_memory()
        wdev = torch.empty(n, dtype=torch.int32, device=dev)

        def e2e_once():
            keys_dev.copy_(host, non_blocking=True)
            wdev.copy_(whost, non_blocking=True)
            r = nsg.window_stats_weighted(keys_dev, wdev, WINDOW, out=outs[0], workspace=ws)
            out_host.copy_(r, non_blocking=True)
        d2h_bytes = WINDOWS_PER_STEP * 9 * 8
    elif world == 1 and nstreams > 1:
        # Consecutive steps overlap: step i runs on lane i mod L (its own stream, device buffers, workspace and
        # pinned result), every step still copies its keys host -> device and its result back; the H2D copies
        # of all lanes share one copy stream, so the PCIe link is never idle while a lane computes.
        lanes = min(nstreams, 2)
        lane_s = [torch.cuda.Stream(dev) for _ in range(lanes)]
        lane_keys = [keys_dev] + [torch.empty(n, dtype=torch.int64, device=dev) for _ in range(lanes - 1)]
        lane_oh = [out_host] + [torch.empty((wps, 9), dtype=torch.int64, pin_memory=True) for _ in range(lanes - 1)]
        lane_i = [0]

        def e2e_once():
            j = lane_i[0] % lanes
            lane_i[0] += 1
            nsg.window_stats_from_host(host, WINDOW, device=dev, keys_dev=lane_keys[j], out=outs[j],
                                       out_host=lane_oh[j], workspace=wss[j], stream=lane_s[j], synchronize=False)
        d2h_bytes = wps * 9 * 8
    else:
        def e2e_once():
            nsg.window_stats_from_host(host, WINDOW, device=dev, keys_dev=keys_dev, out=outs[0], out_host=out_host,
                                       workspace=ws)
            if world > 1:
                gather_window_stats(outs[0], total_windows)
        d2h_bytes = wps * 9 * 8
    for _ in range(2):
        e2e_once()
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s_ in (lane_s if world == 1 and nstreams > 1 and not (vec or anon or trace or wtd) else []):
        s_.wait_event(e0)  # the lanes start after e0
    for _ in range(e2e_steps):
        e2e_once()
    for s_ in (lane_s if world == 1 and nstreams > 1 and not (vec or anon or trace or wtd) else []):
        torch.cuda.current_stream(dev).wait_stream(s_)  # e1 after every lane's last D2H
    e1.record()
    torch.cuda.synchronize(dev)
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=coll_dev)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        e2e_ms = float(tt[0])
    e2e_value = n * world * e2e_steps / (e2e_ms / 1e3)

    if rank == 0:
        peak, peak_src = peaks()
        alg_bytes = n * (BYTES_PER_PACKET + (4 if wtd else 0)) + wps * BYTES_PER_WINDOW_OUT
        if vec:  # + the vectors written: 12 B per link / source / destination, 32 B of IP sets per window
            cnt = outs[0][:, [1, 3, 6]].sum().item()
            alg_bytes += 12 * cnt + 32 * WINDOWS_PER_STEP
        # with overlapping launches (streams > 1) a launch's own duration includes sharing the SMs with its
        # neighbour: the time per launch is the step time
        per_launch_ms = (t_ms / args.steps) if nstreams > 1 else k_avg
        achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9
        cpu = None
        if anon:  # the relabelled src/dst are written: 8 B/packet more
            alg_bytes += n * 8
        if world == 1 and not args.no_cpu_baseline and not (trace or anon):
            cpu = cpu_baseline(dist_, seed)
        spot = None
        if not (trace or anon or wtd):
            last_i = (args.steps - 1) % len(graphs) if graphs else args.steps - 1
            spot = spot_check(dist_, seed, last_rows, first_packet(last_i), sorted({0, wps // 2, wps - 1}))
        suffix = "-vectors" if vec else "-weighted" if wtd else "-trace" if trace else "-anonymize" if anon else ""
        traffic, traffic_src = traffic_per_launch(args.workload + suffix)
        if c4:
            per_gpu = f"{wps} windows x 2^17 packets on this rank (C4 split over {world} ranks)"
        else:
            per_gpu = f"{WINDOWS_PER_STEP} windows x 2^17 packets per GPU per step (C2 batch)"
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s" if wtd else UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if c4 else "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": desc + "; " + per_gpu
                       + ("; outputs: stats + link/source/destination vectors + IP sets" if vec else "")
                       + ("; weighted rows (src, dst, n_packets ~ U[1,8]), unit rows/s" if wtd else "")
                       + ("; WHOLE-TRACE statistics of each step's packets (all ranks' packets together)"
                          if trace else "")
                       + ("; ANONYMISATION of each step's packets (unique, 1 Feistel shuffle round, gather); "
                          "8 B/packet written" if anon else ""),
                       "window": WINDOW, "packets_per_gpu_per_step": n, "parallelism": f"windows sharded dp{world}",
                       "l2": (f"inputs larger than L2: ring of {RING} x {n * 8 >> 20} MiB batches per GPU, no flush"
                              if ring_n > 1 else
                              f"inputs larger than L2: one resident {n * 8 >> 20} MiB block per GPU, no flush" if c4
                              else f"L2-warm: one {n * 8 >> 20} MiB batch reused every step"),
                       "input": "device-resident packed u64 keys (src<<32|dst)",
                       "gather": (f"NCCL all_gather_into_tensor of the [{total_windows}, 9] rows inside the timed region"
                                  if world > 1 else "none (N=1)"),
                       "streams": nstreams,
                       "cuda_graphs": (f"each step replays a captured call ({len(graphs)} graphs: one per ring batch "
                                       "and stream)" if graphs else "no")},
            "value_without_gather": value_no_gather if world > 1 else None,
            "e2e": {"value": e2e_value, "unit": "rows/s" if wtd else UNIT, "h2d_bytes_per_step": n * (12 if wtd else 8),
                    "d2h_bytes_per_step": d2h_bytes, "steps": e2e_steps,
                    "overlap": ("consecutive steps on 2 streams (H2D of one step while the previous one computes)"
                                if world == 1 and nstreams > 1 and not (vec or anon or trace or wtd) else "none")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "frac_vs_nominal_8000": achieved / 8000.0,
                         "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                         "kernel": ("nsg::anon_* (512 MiB bitmap; events around the whole call)" if anon else
                                    "nsg::trace_* (HBM tables; events around the whole call)" if trace else
                                    "nsg::fast_kernel (round-1 kernel; + reset and overflow-check launches: events "
                                    "around the whole call)" if (vec or wtd) else
                                    "nsg::flat::part_kernel + link_kernel + side_kernel: every launch of one call "
                                    "(CUDA events around the whole kernel sequence, excluding the workspace reset)"),
                         "kernel_ms_avg": per_launch_ms,
                         "launch_ms_avg_measured": k_avg,
                         "timing": ("time per call = step time: consecutive calls overlap on "
                                    f"{nstreams} streams" if nstreams > 1 else "CUDA events around each call's kernels"),
                         "algorithmic_bytes_per_launch": alg_bytes},
            "cpu_baseline": cpu,
            "spot_check": spot,
            "clocks": clocks,
            "gpu_launches": launches * args.steps,
            "wall_s_timed_region": wall,
            "diag": diag,
            "build_id": __import__("paper_2509_03653_b200._lib", fromlist=["build_id"]).build_id(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
