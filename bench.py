#!/usr/bin/env python3
"""bench.py — MMA multipath host<->GPU copy on B200 (BASELINE.json metric: "H2D/D2H GB/s per
target GPU vs path count (1/2/4/8) and % of roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mma|reference]
                    [--workload kv|contig] [--bytes B]

One step = one pass of the whole hot path over one batch: the prefix-cache KV fetch of
BASELINE config 3 (131,072 scattered 32 KiB segments = 4 GiB, host pool -> GPU 0 paged
cache) followed by its offload mirror (GPU 0 cache -> host pool), both through the C ABI
(mma_memcpy_h2d_segments / mma_memcpy_d2h_segments) with every path of the set active.
GPU 0 is the target; the k = N path GPUs are GPU 0 (direct) and GPUs 1..N-1 (relays). The
engine is one process driving all paths (§5.1.2 "each process in MMA maintains its
own multipath queue"); under torchrun, ranks > 0 only join the CPU (gloo) barriers so
that no other process time-slices the relay GPUs. Total work is fixed as N grows:
"scaling": "strong". value = bytes moved per step / device time per step (GB/s, 1e9).
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
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "H2D/D2H GB/s per target GPU vs path count (1/2/4/8) and % of roofline"
def _hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except (OSError, ValueError, KeyError):
        return 6650.0, "B200_PROFILING.md fallback"


HBM_PEAK = _hbm_peak()
KNAMES = {0: "zc_copy_kernel", 1: "relay_pull_kernel", 2: "relay_pack_kernel", 3: "zc_dyn_kernel", 4: "zc_bulk_kernel"}
MiB, GiB = 1 << 20, 1 << 30
# PCIe bytes per payload byte of a native copy-engine 4 GiB copy on one B200 link (NVML
# counters, profiles/r01_probe_nvml.json): 256-byte TLPs + DLLPs
CE_PCIE_OVERHEAD = {"h2d": 1.080, "d2h": 1.095}
SEED = 0x4D4D41 + 3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["mma", "reference"], default="mma")
    ap.add_argument("--workload", choices=["kv", "contig", "wake", "contention"], default="kv")
    ap.add_argument("--contention-scale", type=float, default=0.125,
                    help="config 5: fraction of the 17.64 GB TP8 shard (and 4 GiB KV) per GPU")
    ap.add_argument("--bytes", type=int, default=4 * GiB, help="contig workload size")
    ap.add_argument("--tokens", type=int, default=32768, help="kv workload tokens")
    ap.add_argument("--chunk", type=int, default=0, help="chunk bytes (0 = the engine's default)")
    ap.add_argument("--hop", type=int, default=0, help="0 auto, 1 copy engine, 2 SM zero-copy, "
                    "3 copy engine for both relay hops")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--engine-modes", action="store_true",
                    help="N=1: keep the engine's measured mode for the offload (default pins the SM scatter)")
    ap.add_argument("--quick", action="store_true", help="skip baselines (profiling runs)")
    ap.add_argument("--mp", action="store_true",
                    help="multi-process mode (NEXT-4): under torchrun every rank moves its own share of "
                         "the KV fetch/offload on its own GPU (CUDA IPC + shared host memory)")
    ap.add_argument("--loopback", type=int, default=0,
                    help="diagnostic: add loopback relay paths through GPU 0 (exercises the multi-path "
                         "code of the bench on one GPU; the paths share one link)")
    ap.add_argument("--plan", choices=["contiguous", "interleaved", "dynamic"], default=None,
                    help="force the plan mode instead of measuring contiguous vs dynamic")
    ap.add_argument("--modes", default="", help="fix the direct path's mode per direction instead of "
                    "measuring, e.g. 'ce,zc' (profiling runs that must match a bench's choice)")
    return ap.parse_args()


# ------------------------------------------------------------------ distributed ---

class Dist:
    def __init__(self):
        self.rank = int(os.environ.get("RANK", 0))
        self.world = int(os.environ.get("WORLD_SIZE", 1))
        self.local = int(os.environ.get("LOCAL_RANK", 0))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo")   # control plane only: no GPU work on ranks > 0
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def gather_visible(self):
        """Every rank's CUDA_VISIBLE_DEVICES (None = unrestricted), rank order."""
        v = os.environ.get("CUDA_VISIBLE_DEVICES")
        if not self.pg:
            return [v]
        out = [None] * self.world
        self.pg.all_gather_object(out, v)
        return out

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


def engine_gpus(torch):
    """GPUs the engine drives: the visible devices, or more under its virtual-GPU test mode
    (MMA_VGPUS=k: extra engine GPUs on the same devices -- a functional run of
    the multi-path bench on one GPU; its rates are not link rates)"""
    n = torch.cuda.device_count()
    v = int(os.environ.get("MMA_VGPUS", "0") or 0)
    return v if v > n > 0 else n


def cdev(g):
    """torch device of engine GPU g (g itself unless g is a virtual GPU, see engine_gpus)"""
    import torch
    n = torch.cuda.device_count()
    return g % n if n and g >= n else g


# ---------------------------------------------------------------------- clocks ---

class Clocks:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", os.environ.get("MMA_BENCH_SMI_MS", "200"), "-i", ",".join(str(g) for g in sorted({cdev(x) for x in self.gpus}))],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------- workloads ---

def numa_info(torch, gpus):
    """Host NUMA nodes and each path GPU's node (sysfs), for the report."""
    nodes = sorted(p.name for p in Path("/sys/devices/system/node").glob("node[0-9]*"))
    gmap = {}
    for g in gpus:
        try:
            pr = torch.cuda.get_device_properties(cdev(g))
            bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            gmap[str(g)] = int(Path(f"/sys/bus/pci/devices/{bdf}/numa_node").read_text().strip())
        except (OSError, ValueError, AttributeError):
            gmap[str(g)] = None
    return {"nodes": len(nodes), "gpu_node": gmap}


def host_buffer(torch, mma, nbytes):
    """Pinned, mapped host buffer from mma_host_alloc (C8): with more than one NUMA node its
    pages are interleaved across the nodes, so one socket's DRAM does not serve every link.
    Owned by the engine for the life of the process."""
    nodes = len(list(Path("/sys/devices/system/node").glob("node[0-9]*")))
    ptr = mma.host_alloc(nbytes)
    t = torch.from_numpy(mma.host_array(ptr, nbytes))
    how = f"mma_host_alloc, 2 MiB blocks round-robin over {nodes} NUMA nodes" if nodes > 1 else \
        "mma_host_alloc (1 NUMA node: default placement)"
    return t, how


def kv_workload(torch, mma, tokens, dev):
    """Config 3 shapes from mma_inputs.workloads; host pool filled with the seeded pattern
    by the device generator (fill kernel) and copied to the pinned pool."""
    import numpy as np
    from mma_inputs import workloads as W
    shape = W.KVShape() if tokens == 32768 else W.scaled_kv(tokens)
    ho, do, sb, hpool, dbytes = W.kv_segments(shape, SEED)
    host, how = host_buffer(torch, mma, hpool)
    tmp = torch.empty(min(hpool, GiB), dtype=torch.uint8, device=dev)
    for a in range(0, hpool, tmp.numel()):
        n = min(tmp.numel(), hpool - a)
        mma.fill_pattern(tmp, n, SEED, a)
        host[a:a + n].copy_(tmp[:n])
    del tmp
    cache = torch.empty(dbytes, dtype=torch.uint8, device=dev)
    lens = np.full(len(ho), sb, dtype=np.int64)
    fetch = mma.make_segments(host.data_ptr() + ho, cache.data_ptr() + do, lens)
    offload = mma.make_segments(cache.data_ptr() + do, host.data_ptr() + ho, lens)
    # a second request's blocks (disjoint slots and blocks): its offload can overlap the fetch
    ho2, do2, _, _, _ = W.kv_segments(shape, SEED, request=1)
    offload2 = mma.make_segments(cache.data_ptr() + do2, host.data_ptr() + ho2, lens)
    desc = (f"prefix-cache KV fetch + offload (BASELINE config 3): Llama-3-8B bf16 KV, {shape.tokens} tokens, "
            f"{len(ho)} x {sb // 1024} KiB segments (layer, K|V, 16-token block) scattered by a seeded "
            f"permutation in a {hpool / GiB:.0f} GiB pinned pool -> paged device cache")
    return dict(host=host, cache=cache, fetch=fetch, offload=offload, offload2=offload2,
                bytes=int(lens.sum()), ho=ho, do=do,
                sb=sb, desc=desc + f"; pool: {how}", nsegs=len(ho))


def wake_workload(torch, mma, dev):
    """Config 4: vLLM sleep-mode wake of Qwen2.5-14B bf16 (339 tensors, 29,540,067,328 B):
    one pinned backup buffer packed in module order at 256 B, the same layout on the GPU."""
    from mma_inputs import workloads as W
    tensors = W.qwen25_14b_tensors()
    offs, sizes, total = W.packed_layout(tensors)
    host = torch.empty(total, dtype=torch.uint8).pin_memory()
    devbuf = torch.empty(total, dtype=torch.uint8, device=dev)
    mma.fill_pattern(devbuf, total, SEED + 1, 0)
    host.copy_(devbuf)
    desc = (f"vLLM sleep-mode wake + fall-asleep (BASELINE config 4): Qwen2.5-14B bf16, {len(tensors)} "
            f"tensors, {total} B packed at 256 B; one mma_memcpy_h2d / _d2h per tensor")
    return dict(host=host, dev=devbuf, offs=offs, sizes=sizes, bytes=total, desc=desc, wake=True)


def run_half(mma, w, dev_idx, stream, half):
    """half 0 = the step's H2D part (fetch / wake / upload), 1 = its D2H part"""
    if "wake" in w:
        hp, dp = w["host"].data_ptr(), w["dev"].data_ptr()
        for o, n in zip(w["offs"], w["sizes"]):
            if half == 0:
                mma.memcpy_h2d(dp + o, hp + o, n, stream=stream)
            else:
                mma.memcpy_d2h(hp + o, dp + o, n, stream=stream)
    elif "fetch" in w:
        if half == 0:
            mma.memcpy_h2d_segments(*w["fetch"], dev_idx, stream=stream)
        else:
            mma.memcpy_d2h_segments(*w["offload"], dev_idx, stream=stream)
    elif half == 0:
        mma.memcpy_h2d(w["dev"], w["host"], w["bytes"], stream=stream)
    else:
        mma.memcpy_d2h(w["host2"], w["dev"], w["bytes"], stream=stream)


def run_step(mma, w, dev_idx, stream, ev=None):
    if ev: ev[0].record(stream)
    run_half(mma, w, dev_idx, stream, 0)
    if ev: ev[1].record(stream)
    run_half(mma, w, dev_idx, stream, 1)
    if ev: ev[2].record(stream)


# ------------------------------------------------------- hardware byte counters ---

class PcieCounters:
    """NVML's cumulative PCIe byte counters per GPU (RX = into the GPU, TX = out of it;
    SURVEY 8(d): "PCIe bytes per GPU should match the planned bytes per path"). On B200 they
    are 32-bit and wrap every 4 GiB (~75 ms at link rate) and one read takes ~1.3 ms
    (profiles/r01_probe_nvml.json), so a thread samples every GPU continuously and unwraps;
    mark() returns the unwrapped totals after a fresh sample. Used outside the timed region."""

    def __init__(self, torch, gpus):
        import pynvml as N
        N.nvmlInit()
        self.N, self.gpus = N, list(gpus)
        self.h = []
        for g in self.gpus:
            pr = torch.cuda.get_device_properties(cdev(g))
            bdf = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self.h.append(N.nvmlDeviceGetHandleByPciBusId(bdf))
        self.fields = [N.NVML_FI_DEV_PCIE_COUNT_RX_BYTES, N.NVML_FI_DEV_PCIE_COUNT_TX_BYTES]
        self.last = [self._read(h) for h in self.h]
        self.tot = [[0, 0] for _ in self.h]
        self.lock = threading.Lock()
        self.stop_ev = threading.Event()
        self.th = threading.Thread(target=self._loop, daemon=True)
        self.th.start()

    def _read(self, h):
        v = self.N.nvmlDeviceGetFieldValues(h, self.fields)
        if v[0].nvmlReturn or v[1].nvmlReturn:
            raise RuntimeError(f"NVML PCIe counters unsupported ({v[0].nvmlReturn}, {v[1].nvmlReturn})")
        return [int(v[0].value.ullVal), int(v[1].value.ullVal)]

    def nvlink_kib(self):
        """NVML cumulative NVLink data counters per GPU (KiB: [rx, tx]) or None if unsupported
        (relay bytes cross NVLink)."""
        N, out = self.N, []
        for h in self.h:
            v = N.nvmlDeviceGetFieldValues(h, [N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
                                               N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX])
            if v[0].nvmlReturn or v[1].nvmlReturn:
                return None
            out.append([int(v[0].value.ullVal), int(v[1].value.ullVal)])
        return out

    def _pass(self):
        with self.lock:
            for i, h in enumerate(self.h):
                cur = self._read(h)
                for c in range(2):
                    self.tot[i][c] += (cur[c] - self.last[i][c]) % (1 << 32)
                self.last[i] = cur

    def _loop(self):
        while not self.stop_ev.is_set():
            self._pass()
            time.sleep(0.001)

    def mark(self):
        self._pass()
        with self.lock:
            return [list(t) for t in self.tot]

    def close(self):
        self.stop_ev.set()
        self.th.join()


def pcie_hw_check(torch, mma, w, stream, path_gpus, dynamic):
    """One untimed step with the hardware counters running: bytes that entered (H2D) / left
    (D2H) each path GPU over its PCIe link vs the bytes the plan gave that GPU's path."""
    gset = sorted(set(path_gpus))
    cnt = PcieCounters(torch, gset)
    try:
        for g in gset:
            torch.cuda.synchronize(cdev(g))
        out = {"source": "NVML_FI_DEV_PCIE_COUNT_{RX,TX}_BYTES (32-bit, unwrapped by a sampler thread)",
               "note": "counters include TLP/DLLP protocol overhead (~8% H2D, ~9.5% D2H on one B200 link) "
                       "and idle background traffic (~16 KB/ms)"}
        for half, (dname, col) in enumerate((("h2d", 0), ("d2h", 1))):
            mma.reset_stats(0)
            a = cnt.mark()
            na = cnt.nvlink_kib()
            run_half(mma, w, 0, stream, half)
            for g in gset:
                torch.cuda.synchronize(cdev(g))
            b = cnt.mark()
            nb = cnt.nvlink_kib()
            st = mma.get_stats(0)
            paths = mma.get_paths(0, mma.H2D if half == 0 else mma.D2H)
            rows = []
            for i, g in enumerate(gset):
                hw = b[i][col] - a[i][col]
                planned = None if dynamic else sum(int(st["path_bytes"][half][p]) for p, pi in enumerate(paths)
                                                   if pi["gpu"] == g)
                row = {"gpu": g, "planned_bytes": planned, ("rx_bytes" if col == 0 else "tx_bytes"): hw,
                       "ratio": round(hw / planned, 4) if planned else None}
                if na is not None and nb is not None:   # relayed bytes crossing NVLink (KiB counters)
                    row["nvlink_rx_kib"] = nb[i][0] - na[i][0]
                    row["nvlink_tx_kib"] = nb[i][1] - na[i][1]
                rows.append(row)
            out[dname] = rows
        return out
    finally:
        cnt.close()


# --------------------------------------------------------------- cpu baseline ---

def oracle_sample(k_paths, nsegs_sample=16384, reps=1, min_seconds=0.0):
    """The oracle's threaded mover (1 thread for the direct path + 2 per relay ring) on a
    bounded sample of the KV workload: the first `nsegs_sample` segments, gathered from
    their scattered slots of a pinned-pool-sized host buffer into a packed host 'cache',
    then scattered back (offload); repeated `reps` times or until `min_seconds` of CPU work
    (at most 30 repetitions). Returns (GB/s of the median repetition, threads, sample
    description, bytes per repetition, seconds of the median repetition)."""
    import numpy as np
    import oracle
    from mma_inputs import workloads as W
    shape = W.KVShape()
    ho, do, sb, hpool, dbytes = W.kv_segments(shape, SEED)
    ho = ho[:nsegs_sample]
    span = int(ho.max()) + sb
    pool = np.empty(span, dtype=np.uint8)
    pool[::4096] = 1                                   # touch the pages
    cache = np.empty(nsegs_sample * sb, dtype=np.uint8)
    cache[::4096] = 1
    dofs = np.arange(nsegs_sample, dtype=np.int64) * sb
    lens = np.full(nsegs_sample, sb, dtype=np.int64)
    B = int(lens.sum())
    C = 4 * MiB
    bw = [1] * k_paths
    rc, path, _, _ = oracle.plan(bw, B, C, 0, oracle.CONTIG)
    f_segs, n = oracle.segments_from_arrays(pool.ctypes.data + ho, cache.ctypes.data + dofs, lens)
    o_segs, _ = oracle.segments_from_arrays(cache.ctypes.data + dofs, pool.ctypes.data + ho, lens)
    times = []
    while len(times) < max(reps, 1) or (sum(times) < min_seconds and len(times) < 30):
        t0 = time.perf_counter()
        assert oracle.move(f_segs, n, C, bw, path, S=4, exec_mode=oracle.THREADED) == 0
        assert oracle.move(o_segs, n, C, bw, path, S=4, exec_mode=oracle.THREADED) == 0
        times.append(time.perf_counter() - t0)
    med = statistics.median(times)
    threads = 1 + 2 * (k_paths - 1)
    desc = (f"oracle threaded mover (oracle/mma_oracle.c, exec=threaded, {k_paths}-path plan), first "
            f"{nsegs_sample} of 131072 KV segments ({B / MiB:.0f} MiB) fetched into a packed host buffer "
            f"and offloaded back, host memory only; {len(times)} repetitions ({sum(times):.1f} s), median")
    return 2 * B / med / 1e9, threads, desc, 2 * B, med


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(k_paths, nsegs_sample=32768, seconds_per_leg=6.0):
    """the cpu_baseline object: the oracle mover at T = the k-path thread set and at T ~ nproc"""
    nproc = os.cpu_count() or 1
    legs = []
    for kk in dict.fromkeys([k_paths, max(1, (nproc + 1) // 2)]):
        g, threads, desc, _, _ = oracle_sample(kk, nsegs_sample=nsegs_sample, reps=5, min_seconds=seconds_per_leg)
        legs.append({"paths": kk, "threads": threads, "gbps": round(g, 3), "sample": desc})
    head = legs[0]
    return {"value": head["gbps"], "unit": "GB/s", "cores": head["threads"], "kind": "oracle",
            "sample": head["sample"], "legs": legs, "nproc": nproc, "cpu_model": cpu_model(),
            "note": "value/cores = the leg with the bench's own path count; the other leg runs the same oracle "
                    "with (nproc + 1) // 2 paths so its threads (1 + 2 per relay) fill the host's cores"}


def run_reference(args, dist):
    """--impl reference: the oracle as it stands on the host cores (the base contract's
    reference arm for this tier); rank 0 only."""
    if dist.rank != 0:
        return
    import oracle
    oracle.build()
    k = max(1, args.gpus)
    times = []
    gbps = None
    for i in range(args.warmup + args.steps):
        g, threads, desc, nbytes, dt = oracle_sample(k, nsegs_sample=8192)
        if i >= args.warmup:
            times.append(dt)
    dt = statistics.median(times)
    gbps = nbytes / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbps, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "prefix-cache KV fetch + offload (BASELINE config 3), bounded sample",
                   "paths": k},
        "cpu_baseline": {"value": round(gbps, 3), "unit": "GB/s", "cores": threads, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": round(gbps, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- roofline ---

def pcie_rate(torch, g, nbytes=GiB, reps=8):
    """Solo native cudaMemcpyAsync GB/s of GPU g's PCIe link per direction (the roofline's
    PCIe term and R(1))."""
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{cdev(g)}")
    s = torch.cuda.Stream(device=cdev(g))
    out = {}
    for name in ("h2d", "d2h"):
        best = 1e9
        with torch.cuda.device(cdev(g)), torch.cuda.stream(s):
            for _ in range(reps):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(s)
                if name == "h2d":
                    d.copy_(h, non_blocking=True)
                else:
                    h.copy_(d, non_blocking=True)
                b.record(s)
                b.synchronize()
                best = min(best, a.elapsed_time(b))
        out[name] = nbytes / best / 1e6
    del h, d
    return out


def dram_read_rate(torch, nbytes=2 * GiB, reps=3):
    """Host DRAM read GB/s with every core (torch CPU reduction over an int64 buffer)."""
    t = torch.ones(nbytes // 8, dtype=torch.int64)
    threads = torch.get_num_threads()
    torch.set_num_threads(os.cpu_count() or 1)     # torchrun sets OMP_NUM_THREADS=1
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        t.sum()
        best = min(best, time.perf_counter() - t0)
    torch.set_num_threads(threads)
    del t
    return nbytes / best / 1e9


def conc_rate(torch, gpus, per_gpu=512 * MiB, reps=3):
    """R_conc(k): k concurrent plain cudaMemcpyAsync, each path GPU moving its own slice of
    one pinned buffer: the achievable hop-1 ceiling of this box, exposing
    shared switch uplinks and the host-memory ceiling."""
    k = len(gpus)
    host = torch.empty(k * per_gpu, dtype=torch.uint8).pin_memory()
    devs = [torch.empty(per_gpu, dtype=torch.uint8, device=f"cuda:{cdev(g)}") for g in gpus]
    streams = [torch.cuda.Stream(device=cdev(g)) for g in gpus]
    out = {}
    for name in ("h2d", "d2h"):
        best = 1e9
        for _ in range(reps):
            for g in gpus:
                torch.cuda.synchronize(cdev(g))
            t0 = time.perf_counter()
            for i, g in enumerate(gpus):
                with torch.cuda.device(cdev(g)), torch.cuda.stream(streams[i]):
                    sl = host[i * per_gpu:(i + 1) * per_gpu]
                    if name == "h2d":
                        devs[i].copy_(sl, non_blocking=True)
                    else:
                        sl.copy_(devs[i], non_blocking=True)
            for s in streams:
                s.synchronize()
            best = min(best, time.perf_counter() - t0)
        out[name] = k * per_gpu / best / 1e9
    del host, devs
    return out


def nvlink_rate(torch, target, relays, per_gpu=512 * MiB, reps=3):
    """NVLink ingress into / egress out of the target from every relay at once (SURVEY 8(d):
    the roofline term PCIe[d] + NVLinkIn[d]): each relay's copy engine moves its own buffer
    to (from) the target concurrently; wall time around the whole set, best of reps."""
    if not relays:
        return None
    tgt = [torch.empty(per_gpu, dtype=torch.uint8, device=f"cuda:{cdev(target)}") for _ in relays]
    src = [torch.empty(per_gpu, dtype=torch.uint8, device=f"cuda:{cdev(g)}") for g in relays]
    streams = [torch.cuda.Stream(device=cdev(g)) for g in relays]
    out = {}
    for name in ("ingress", "egress"):
        best = 1e9
        for _ in range(reps):
            for g in [target] + list(relays):
                torch.cuda.synchronize(cdev(g))
            t0 = time.perf_counter()
            for i, g in enumerate(relays):
                with torch.cuda.device(cdev(g)), torch.cuda.stream(streams[i]):
                    if name == "ingress":
                        tgt[i].copy_(src[i], non_blocking=True)
                    else:
                        src[i].copy_(tgt[i], non_blocking=True)
            for st in streams:
                st.synchronize()
            best = min(best, time.perf_counter() - t0)
        out[name] = len(relays) * per_gpu / best / 1e9
    del tgt, src
    return out


def timeline_summary(path):
    """Per-GPU busy time and GPU concurrency of one traced step (engine Chrome trace)."""
    ev = json.load(open(path))["traceEvents"]
    if not ev:
        return None
    per_gpu = {}
    for e in ev:
        per_gpu.setdefault(e["pid"], []).append((e["ts"], e["ts"] + e["dur"]))
    t0 = min(s for v in per_gpu.values() for s, _ in v)
    t1 = max(e for v in per_gpu.values() for _, e in v)
    pts = sorted({x for v in per_gpu.values() for s in v for x in s})
    weighted = 0.0
    for a, b in zip(pts, pts[1:]):
        m = (a + b) / 2
        weighted += (b - a) * sum(any(s <= m < e for s, e in v) for v in per_gpu.values())
    busy = {g: round(sum(e - s for s, e in _merge(v)), 1) for g, v in sorted(per_gpu.items())}
    return {"span_us": round(t1 - t0, 1), "busy_us": busy, "mean_gpus_busy": round(weighted / max(t1 - t0, 1e-9), 2),
            "spans": len(ev)}


def _merge(iv):
    out = []
    for s, e in sorted(iv):
        if out and s <= out[-1][1]:
            out[-1][1] = max(out[-1][1], e)
        else:
            out.append([s, e])
    return out


def ncu_traffic(direction, kernel):
    """dram bytes per launch of the dominant kernel from the committed ncu capture
    (profiles/ncu_summary.json), or None when that kernel was not captured."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists() and kernel in ("zc_copy_kernel", "zc_bulk_kernel"):
        try:
            e = json.loads(p.read_text()).get("kernels", {}).get(f"{kernel}/{direction}")
            return e.get("dram_bytes_per_launch") if e else None
        except (ValueError, AttributeError):
            return None
    return None


# ----------------------------------------------------------------------- main ---

def run_mp(args, dist, torch, mma):
    """--mp: one process per GPU. Rank 0 owns the target cache (GPU 0) and
    exports it by CUDA IPC; the host pool is named shared memory pinned by every rank; each
    rank moves its share of every fetch and offload with the zero-copy kernel on its own GPU
    -- the chunks the common contiguous plan gives its path, or the units it claims from a
    cursor in GPU 0's memory (dynamic), whichever measured faster. Each phase is bracketed by
    gloo barriers; a phase's time is the max over ranks of the rank's own CUDA-event time."""
    import numpy as np
    from mma_inputs import workloads as W
    rank, world = dist.rank, dist.world
    ngpu = torch.cuda.device_count()
    dev = dist.local if ngpu > 1 else 0
    torch.cuda.set_device(dev)
    shape = W.KVShape() if args.tokens == 32768 else W.scaled_kv(args.tokens)
    ho, do, sb, hpool, dbytes = W.kv_segments(shape, SEED)
    lens = np.full(len(ho), sb, dtype=np.int64)
    Bytes = int(lens.sum())
    name = f"bench_{os.environ.get('MASTER_PORT', '0')}"
    cfg = mma.default_config()
    cfg.debug_log = 0
    mma.init(cfg)
    if rank == 0:
        pool = mma.shared_host_alloc(name, hpool, True)
        pt = torch.from_numpy(mma.host_array(pool, hpool))
        tmp = torch.empty(min(hpool, GiB), dtype=torch.uint8, device="cuda")
        for a in range(0, hpool, tmp.numel()):
            n = min(tmp.numel(), hpool - a)
            mma.fill_pattern(tmp, n, SEED, a)
            pt[a:a + n].copy_(tmp[:n])
        del tmp
        cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
        ctr = torch.zeros(32, dtype=torch.int64, device="cuda")
        obj = [(mma.ipc_export(cache), mma.ipc_export(ctr))]
    else:
        obj = [None]
    dist.barrier()
    dist.pg.broadcast_object_list(obj, src=0)
    (hd, od), (hc, oc) = obj[0]
    if rank == 0:
        cptr, kptr = cache.data_ptr(), ctr.data_ptr()
    else:
        pool = mma.shared_host_alloc(name, hpool, False)
        cptr, kptr = mma.ipc_open(hd, od, dev), mma.ipc_open(hc, oc, dev)
    fetch = mma.make_segments(pool + ho, cptr + do, lens)
    offload = mma.make_segments(cptr + do, pool + ho, lens)
    C, claim = 8 * MiB, 256 << 10
    rc, plan, _ = mma.plan_chunks([1] * world, [0] + [1] * (world - 1), Bytes, C, 0, 0)
    s = torch.cuda.Stream()

    def phase(segs, dynamic):
        if dynamic and rank == 0:
            ctr.zero_()
            torch.cuda.synchronize()
        dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        if dynamic:
            mma.copy_claim_segments(*segs, claim, kptr, kptr + 8, rank, dev, stream=s)
        else:
            mma.copy_share_segments(*segs, C, plan, rank, dev, stream=s)
        b.record(s)
        b.synchronize()
        return dist.max(a.elapsed_time(b))

    def step(dynamic):
        return phase(fetch, dynamic) + phase(offload, dynamic)

    for _ in range(args.warmup):
        step(False)
    t_plan = statistics.median(step(False) for _ in range(2))
    t_dyn = statistics.median(step(True) for _ in range(2))
    dynamic = t_dyn < t_plan
    verify = None
    if rank == 0:
        cache.zero_()
        torch.cuda.synchronize()
    phase(fetch, dynamic)
    if rank == 0:
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        mma.verify_segments(cache.data_ptr() + do, ho, lens, SEED, cnt)
        torch.cuda.synchronize()
        verify = {"mismatched_bytes": int(cnt.item()), "checked_bytes": Bytes, "on": "device (C4)"}
    mma.set_kernel_timing(True)
    times = [step(dynamic) for _ in range(args.steps)]
    kt = mma.kernel_times()
    mma.set_kernel_timing(False)
    ms_step = statistics.mean(times)
    value = 2 * Bytes / (ms_step * 1e-3) / 1e9
    err = mma.get_last_error()
    dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "prefix-cache KV fetch + offload (BASELINE config 3), multi-process mode",
                       "paths": world, "parallelism": "one process per GPU; rank r moves path r's share on "
                       "its own GPU (CUDA IPC destination, shared pinned host pool); phase time = max over ranks",
                       "plan": {"contiguous_ms": round(t_plan, 3), "dynamic_ms": round(t_dyn, 3),
                                "chosen": "dynamic" if dynamic else "contiguous"},
                       "gpus_visible_per_rank": ngpu},
            "gpu_launches": len(kt), "verify": verify, "engine_error": err,
            "e2e": None, "roofline": None, "cpu_baseline": None,
            "note": "rank-0 line of the multi-process mode; the default (single-process) bench carries "
                    "roofline, e2e and cpu_baseline",
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    if rank != 0:
        mma.ipc_close(cptr)
        mma.ipc_close(kptr)
        mma.shared_host_free(pool)
    dist.barrier()
    if rank == 0:
        mma.shared_host_free(pool, name)


def widen_visible(dist, visible_sets):
    """Rank 0 drives every path GPU: if each rank was given only its own device, widen rank
    0's view to the union of the job's devices (gathered before any CUDA call)."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if dist.world <= 1 or not visible_sets or any(v is None for v in visible_sets):
        return None
    union = []
    for v in visible_sets:
        for x in (y.strip() for y in v.split(",")):
            if x and x not in union:
                union.append(x)
    if len(union) > len([x for x in (vis or "").split(",") if x.strip()]):
        os.environ["CUDA_VISIBLE_DEVICES"] = ",".join(union)
        return f"CUDA_VISIBLE_DEVICES={vis} widened for rank 0 to the job's devices {','.join(union)}"
    return None


def run_contention(args, dist, torch, mma, visible_sets):
    """BASELINE config 5: every path GPU reloads its Llama-3-70B TP8 weight shard at once
    (one contiguous H2D per GPU, each on its own stream) while GPUs 0 and 1 also fetch a
    prefix-cache KV table -- all through one engine, whose backlog ledger plans each call
    against the bytes already queued on every link and keeps a GPU with its own direct work
    from relaying (NEXT-1). Reported: aggregate GB/s (wall clock around issue + completion of
    the whole batch), per-target completion, vs the same batch with native copies. The bar
    is no regression vs native (relays should only use spare capacity)."""
    import numpy as np
    from mma_inputs import workloads as W
    if dist.rank != 0:
        dist.barrier()
        dist.barrier()
        dist.max(0.0)
        dist.barrier()
        return
    widen_visible(dist, visible_sets)
    k = max(1, min(args.gpus, engine_gpus(torch)))
    gpus = list(range(k))
    shard = int(17_640_734_720 * args.contention_scale) // 4096 * 4096
    hosts, devs, streams = [], [], []
    for g in gpus:
        p = mma.host_alloc(shard)
        hosts.append(p)
        devs.append(torch.empty(shard, dtype=torch.uint8, device=f"cuda:{cdev(g)}"))
        streams.append(torch.cuda.Stream(device=cdev(g)))
    tokens = max(256, int(32768 * args.contention_scale) // 16 * 16)
    kvs = []
    for g in gpus[:2]:
        shape = W.scaled_kv(tokens)
        ho, do, sb, hpool, dbytes = W.kv_segments(shape, SEED + g)
        pool = mma.host_alloc(hpool)
        cache = torch.empty(dbytes, dtype=torch.uint8, device=f"cuda:{cdev(g)}")
        lens = np.full(len(ho), sb, dtype=np.int64)
        kvs.append((g, mma.make_segments(pool + ho, cache.data_ptr() + do, lens), int(lens.sum()), cache,
                    torch.cuda.Stream(device=cdev(g))))
    total = shard * k + sum(x[2] for x in kvs)

    reload_segs = [mma.make_segments([hosts[i]], [devs[i].data_ptr()], [shard]) for i in range(k)]

    def batch(joint):
        for g in gpus:
            torch.cuda.synchronize(cdev(g))
        t0 = time.perf_counter()
        if joint:      # one joint plan for the whole batch (mma_memcpy_multi, NEXT-1)
            mma.memcpy_multi([(mma.H2D, g, reload_segs[i], streams[i]) for i, g in enumerate(gpus)] +
                             [(mma.H2D, g, segs, s) for g, segs, nb, cache, s in kvs])
        else:          # one call per transfer, each planned against the ledger's backlog
            for i, g in enumerate(gpus):      # one segment = the contiguous copy into GPU g
                mma.memcpy_h2d_segments(*reload_segs[i], g, stream=streams[i])
            for g, segs, nb, cache, s in kvs:
                mma.memcpy_h2d_segments(*segs, g, stream=s)
        for g in gpus:
            torch.cuda.synchronize(cdev(g))
        return time.perf_counter() - t0

    def measure(native, joint=False):
        cfg = mma.default_config()
        cfg.debug_log = 0
        if native:
            cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = (1 << 64) - 1
        mma.init(cfg)
        for _ in range(max(1, args.warmup)):
            batch(joint)
        return statistics.median(batch(joint) for _ in range(args.steps))

    t_native = measure(True)
    t_calls = measure(False)
    for g in gpus:
        mma.reset_stats(g)
    t_mma = measure(False, joint=True)
    relay = sum(mma.get_stats(g)["relay_bytes"] for g in gpus)
    assert mma.get_last_error() == 0
    dist.barrier()
    dist.barrier()
    t_mma = dist.max(t_mma)
    dist.barrier()
    line = {"metric": METRIC, "value": round(total / t_mma / 1e9, 3), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_mma * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": f"contention (BASELINE config 5): {k} GPU(s) each reload a Llama-3-70B TP8 "
                                   f"bf16 shard x{args.contention_scale} ({shard} B) at once while GPUs "
                                   f"{[x[0] for x in kvs]} fetch {tokens}-token KV; aggregate over the batch",
                       "paths_per_target": k},
            "native": {"gbps": round(total / t_native / 1e9, 3), "ms": round(t_native * 1e3, 3)},
            "per_call_ledger": {"gbps": round(total / t_calls / 1e9, 3), "ms": round(t_calls * 1e3, 3),
                                "what": "one call per transfer, each planned against the ledger's backlog"},
            "speedup_vs_native": round(t_native / t_mma, 3),
            "relay_bytes_per_batch": relay // (max(1, args.warmup) + args.steps),
            "note": "value: the whole batch under one joint plan (mma_memcpy_multi: per-GPU queues, direct "
                    "path first, longest queue relayed first, P:549-574); wall clock around issue + "
                    "completion on every GPU"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    dist = Dist()
    if args.impl == "reference":
        run_reference(args, dist)
        dist.close()
        return
    import torch
    import paper_2512_16056_b200 as mma

    if args.mp and dist.world > 1:
        run_mp(args, dist, torch, mma)
        dist.close()
        return
    visible_sets = dist.gather_visible()
    if args.workload == "contention":
        run_contention(args, dist, torch, mma, visible_sets)
        dist.close()
        return

    if dist.rank != 0:
        # ranks > 0: no GPU work of their own; their GPUs serve as rank 0's relay paths
        dist.barrier()      # setup done
        dist.barrier()      # before timed region
        dist.max(0.0)
        dist.barrier()      # after
        dist.close()
        return

    vis_note = widen_visible(dist, visible_sets)
    ngpu_vis = engine_gpus(torch)
    k = max(1, min(args.gpus, ngpu_vis))
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream(device=0)
    early = mma.default_config()
    early.numa_mode = 3                      # host buffers in 2 MiB blocks round-robin over the nodes
    mma.init(early)

    if args.workload == "kv":
        w = kv_workload(torch, mma, args.tokens, dev)
    elif args.workload == "wake":
        w = wake_workload(torch, mma, dev)
    else:
        B = args.bytes
        host = torch.empty(B, dtype=torch.uint8).pin_memory()
        tmp = torch.empty(B, dtype=torch.uint8, device=dev)
        mma.fill_pattern(tmp, B, SEED, 0)
        host.copy_(tmp)
        w = dict(host=host, host2=torch.empty(B, dtype=torch.uint8).pin_memory(), dev=tmp, bytes=B,
                 desc=f"single {B / MiB:.0f} MiB contiguous H2D + D2H (BASELINE config 2 point)")
    nbytes_step = 2 * w["bytes"]

    def configure(relays):
        cfg = mma.default_config()
        if args.chunk:
            cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = args.chunk
        cfg.npaths = len(relays) if relays else 1
        for i, g in enumerate(relays or [0]):
            cfg.path_gpus[i] = g          # [0] alone = no relay candidates (self is skipped)
        cfg.loopback_relays = args.loopback
        cfg.plan_mode = 0
        cfg.hop_mode[0] = cfg.hop_mode[1] = args.hop
        cfg.debug_log = 0
        cfg.numa_mode = 3
        mma.init(cfg)
        return cfg

    thresholds = {}
    policy = {}

    def offload_rate(mode, calls=3):
        """D2H rate of the workload's offload with the single path pinned to `mode`: `calls`
        offloads enqueued back to back after a warm-up call (as the timed region runs them)"""
        mma.set_path_modes(0, mma.D2H, [mode])
        mma.memcpy_d2h_segments(*w["offload"], 0, stream=stream)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(calls):
            mma.memcpy_d2h_segments(*w["offload"], 0, stream=stream)
        b.record(stream)
        b.synchronize()
        return round(calls * w["bytes"] / (a.elapsed_time(b) * 1e-3) / 1e9, 2)

    def prepare(relays):
        """engine config, per-path mode/bandwidth by measurement, warm-up and a device-side
        check of the bench's own launch configuration (all outside the timed region)"""
        cfg = configure(relays)
        if args.modes:
            m = {"ce": mma.HOP_CE, "zc": mma.HOP_ZC, "ce_p2p": mma.HOP_CE_P2P, "push": mma.HOP_PUSH}
            h, d = (m[x] for x in args.modes.split(","))
            mma.set_path_modes(0, mma.H2D, [h] * len(mma.get_paths(0, mma.H2D)))
            mma.set_path_modes(0, mma.D2H, [d] * len(mma.get_paths(0, mma.D2H)))
        elif args.hop == 0:
            if "fetch" in w:
                mma.tune_segments(*w["fetch"], 0, mma.H2D, stream=stream, reps=2)
                mma.tune_segments(*w["offload"], 0, mma.D2H, stream=stream, reps=2)
            else:
                mma.calibrate(0, mma.H2D, min(w["bytes"], GiB))
                mma.calibrate(0, mma.D2H, min(w["bytes"], GiB))
            if len(mma.get_paths(0, mma.D2H)) == 1 and "fetch" in w and not args.engine_modes:
                # N = 1 policy (DESIGN 6.1): with one path the copy engine in host-address order
                # can beat the SM scatter on the offload; the line times the repo's kernel path
                # (a7/a10) and reports both rates from this run
                tuned_d2h = mma.get_paths(0, mma.D2H)
                ce, zc = offload_rate(mma.HOP_CE), offload_rate(mma.HOP_ZC)
                policy.update({"d2h_single_path": "SM zero-copy scatter (pinned for the line)",
                               "measured_choice": {1: "ce", 2: "zc"}.get(tuned_d2h[0]["seg_mode"], "?"),
                               "d2h_ce_host_order_gbps": ce, "d2h_zc_gbps": zc,
                               "note": "copy-engine DMAs (one cudaMemcpyAsync per block) run in host-address order (cfg.host_order); "
                                       "--engine-modes times the engine's own measured choice"})
            if len(mma.get_paths(0, mma.H2D)) > 1 and "fetch" not in w:
                # the fallback threshold is the measured native/multipath break-even of
                # a contiguous copy (a single path needs none; the 4 GiB KV calls are far above it)
                for name, dv in (("h2d", mma.H2D), ("d2h", mma.D2H)):
                    thr, found = mma.tune_threshold(0, dv, 256 * MiB)
                    thresholds[name] = thr if found else f"no break-even up to 256 MiB (kept {thr})"
        for _ in range(args.warmup):
            run_step(mma, w, 0, stream)
        stream.synchronize()
        verify = None
        if not args.no_verify and "fetch" in w:
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            torch.cuda.synchronize(0)
            with torch.cuda.stream(stream):
                w["cache"].zero_()                      # ordered before the fetch on `stream`
            mma.memcpy_h2d_segments(*w["fetch"], 0, stream=stream)
            mma.verify_segments(w["cache"].data_ptr() + w["do"], w["ho"], [w["sb"]] * w["nsegs"], SEED, cnt,
                                stream=stream)
            stream.synchronize()
            verify = {"mismatched_bytes": int(cnt.item()), "checked_bytes": w["bytes"], "on": "device (C4)"}
            if verify["mismatched_bytes"]:
                raise RuntimeError(f"multipath copy verification failed: {verify}")
        if not args.no_verify and "wake" in w:
            cnt = torch.zeros(1, dtype=torch.int64, device=dev)
            torch.cuda.synchronize(0)
            with torch.cuda.stream(stream):
                w["dev"].zero_()
            run_step(mma, w, 0, stream)               # wake (H2D) then fall asleep (D2H)
            mma.verify_pattern(w["dev"], w["bytes"], SEED + 1, 0, cnt, stream=stream)
            stream.synchronize()
            verify = {"mismatched_bytes": int(cnt.item()), "checked_bytes": w["bytes"], "on": "device (C4)"}
            if verify["mismatched_bytes"]:
                raise RuntimeError(f"multipath copy verification failed: {verify}")
        if mma.get_last_error():
            raise RuntimeError(f"sticky engine error {mma.get_last_error()}")
        return cfg, verify

    multipath_error = None
    try:
        cfg, verify = prepare(list(range(1, k)))
    except Exception as ex:  # noqa: BLE001 - report, then retry without relay kernels, then direct
        multipath_error = f"{type(ex).__name__}: {ex}"
        print(f"multipath setup failed ({multipath_error}); retrying with zero-copy paths only", file=sys.stderr)
        mma.finalize()
        saved_modes = args.modes
        try:
            if k > 1 and "fetch" in w:   # the one-hop zero-copy relays need no ring and no flag
                args.modes = "zc,zc"
                cfg, verify = prepare(list(range(1, k)))
                multipath_error += " (retried: every path zero-copy)"
            else:
                raise RuntimeError("no zero-copy retry for this workload")
        except Exception as ex2:  # noqa: BLE001 - measure the direct path alone
            args.modes = saved_modes
            multipath_error += f"; retry failed ({type(ex2).__name__}: {ex2}); direct path only"
            print(f"falling back to the direct path ({multipath_error})", file=sys.stderr)
            mma.finalize()
            k = 1
            cfg, verify = prepare([])
    paths = mma.get_paths(0, mma.H2D)
    path_gpus = [p["gpu"] for p in paths]
    fallback_cfg = {"h2d": int(cfg.fallback_bytes[0]), "d2h": int(cfg.fallback_bytes[1])}
    try:
        topology = mma.get_topology()   # P2P matrix, NUMA node, copy engines per GPU
    except Exception as ex:  # noqa: BLE001 - evidence only
        topology = {"error": str(ex)}
    tuned = {"h2d": mma.get_paths(0, mma.H2D), "d2h": mma.get_paths(0, mma.D2H)}
    # each path's rate alone (mode choice) and with every path active (planner)
    calib = {d: mma.get_calibration(0, dv, scattered="fetch" in w)
             for d, dv in (("h2d", mma.H2D), ("d2h", mma.D2H))}

    # planned (contiguous, measured bandwidth split) vs GPU-driven dynamic pull: chosen by
    # measurement when more than one path exists (dynamic applies to all-zero-copy sets)
    plan_choice = {"chosen": "contiguous"}
    if len(path_gpus) > 1 and not args.plan:
        def step_ms(mode):
            mma.set_plan_mode(mode)
            run_step(mma, w, 0, stream)
            stream.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(2):
                run_step(mma, w, 0, stream)
            b.record(stream)
            b.synchronize()
            return a.elapsed_time(b) / 2
        t_static, t_dyn = step_ms(0), step_ms(2)
        plan_choice = {"contiguous_ms": round(t_static, 3), "dynamic_ms": round(t_dyn, 3),
                       "chosen": "dynamic" if t_dyn < t_static else "contiguous"}
        mma.set_plan_mode(2 if t_dyn < t_static else 0)
    elif args.plan:
        mma.set_plan_mode({"contiguous": 0, "interleaved": 1, "dynamic": 2}[args.plan])
        plan_choice = {"chosen": args.plan, "forced": True}

    # roofline terms (solo PCIe per path GPU), measured before the timed region
    pcie = {g: pcie_rate(torch, g) for g in path_gpus}
    R_h2d = sum(pcie[g]["h2d"] for g in path_gpus)
    R_d2h = sum(pcie[g]["d2h"] for g in path_gpus)

    # ---- timed region
    mma.reset_stats(0)
    mma.set_kernel_timing(True)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clocks = Clocks(path_gpus)
    dist.barrier()
    dist.barrier()
    for g in path_gpus:
        torch.cuda.synchronize(cdev(g))
    clocks.start()
    time.sleep(0.3)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    import resource
    ru0, w0 = resource.getrusage(resource.RUSAGE_SELF), time.perf_counter()
    t_start.record(stream)
    for i in range(args.steps):
        run_step(mma, w, 0, stream, evs[i])
    t_end.record(stream)
    for g in path_gpus:
        torch.cuda.synchronize(cdev(g))
    ru1, w1 = resource.getrusage(resource.RUSAGE_SELF), time.perf_counter()
    clk = clocks.stop()
    # host CPU the engine needs (the paper's Fig 13 / P:934: two busy threads per GPU cost
    # 822% CPU at 8 GPUs); ours has no thread in the per-chunk loop, only the enqueue
    cpu_s = (ru1.ru_utime - ru0.ru_utime) + (ru1.ru_stime - ru0.ru_stime)
    host_cpu = {"process_cpu_percent": round(100 * cpu_s / max(1e-9, w1 - w0), 1),
                "what": "process user+system CPU over the timed region / wall time; includes the host "
                        "thread spinning in cudaStreamSynchronize (torch's default sync) -- the engine's "
                        "own share is engine.enqueue_cpu_percent"}
    ktimes = mma.kernel_times()
    mma.set_kernel_timing(False)
    ms_total = t_start.elapsed_time(t_end)
    ms_total = dist.max(ms_total)
    dist.barrier()
    st = mma.get_stats(0)
    assert mma.get_last_error() == 0
    ms_step = ms_total / args.steps
    value = nbytes_step / (ms_step * 1e-3) / 1e9
    h2d_ms = statistics.median(evs[i][0].elapsed_time(evs[i][1]) for i in range(args.steps))
    d2h_ms = statistics.median(evs[i][1].elapsed_time(evs[i][2]) for i in range(args.steps))
    h2d_gbps = w["bytes"] / (h2d_ms * 1e-3) / 1e9
    d2h_gbps = w["bytes"] / (d2h_ms * 1e-3) / 1e9

    # dominant kernel: the (kind, direction, path, device) group with the largest total
    # launch time in the timed region; its bytes per launch / its mean launch duration,
    # against the solo PCIe rate of the link(s) it is bound by
    groups = {}
    for kt in ktimes:
        groups.setdefault((kt["kind"], kt["dir"], kt["path"], kt["dev"]), []).append(kt["ms"])
    kinds = sorted({kt["kind"] for kt in ktimes})
    roof = None
    if groups:
        (kind, kdir, kpath, kdev), ms_list = max(groups.items(), key=lambda kv: sum(kv[1]))
        dname = "h2d" if kdir == 0 else "d2h"
        pinfo = tuned[dname]

        def eff_mode(pi):
            m = pi["seg_mode"] if ("fetch" in w and pi["seg_mode"] >= 0) else pi["mode"]
            return m if m else (2 if "fetch" in w else 1)
        if kind == 3:         # dynamic pull: every path's kernel serves the same call
            moved = w["bytes"] * args.steps
            ms_list = [(h2d_ms if kdir == 0 else d2h_ms)] * args.steps
            peak = sum(pcie[g][dname] for g in path_gpus)
        elif kpath == 255:    # one relay kernel serves every copy-engine ring of the call
            ring_paths = [i for i, pi in enumerate(pinfo) if pi["kind"] == 1 and eff_mode(pi) in (1, 4)]
            moved = sum(st["path_bytes"][kdir][i] for i in ring_paths)
            peak = sum(pcie[pinfo[i]["gpu"]][dname] for i in ring_paths)
        else:
            moved = st["path_bytes"][kdir][kpath]
            peak = pcie[pinfo[kpath]["gpu"]][dname]
        per_launch = moved // max(1, len(ms_list))
        k_ms = statistics.mean(ms_list)
        achieved = per_launch / (k_ms * 1e-3) / 1e9
        roof = {"bound": "pcie", "achieved": round(achieved, 2), "peak": round(peak, 2), "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(dname, KNAMES[kind]),
                "kernel": KNAMES[kind] + (" (all paths of the call; duration = the call's events)" if kind == 3 else ""),
                "direction": dname, "path": kpath, "device": kdev, "launches": len(ms_list),
                "bytes_per_launch": per_launch, "launch_ms": round(k_ms, 3),
                "share_of_step": round(sum(ms_list) / ms_total, 4),
                "peak_source": f"measured in this run: solo native cudaMemcpyAsync 1 GiB {dname.upper()} "
                               "over the PCIe link(s) this kernel's bytes cross (the roofline's PCIe "
                               "term, SURVEY 8(d)); HBM is not the bound of a host<->device copy",
                "hbm_reference": {"peak_gbps": HBM_PEAK[0], "source": HBM_PEAK[1],
                                  "frac": round(achieved / HBM_PEAK[0], 5) if HBM_PEAK[0] else None,
                                  "note": "the same bytes against HBM copy bandwidth, for context"}}

    # path-level roofline: R(k) = min(sum of the used links' solo PCIe rates,
    # host DRAM), DRAM taken as the lower bound max(all-core CPU read, R_conc(k)); R_conc(k)
    # (k plain copies at once) reported beside it. NVLink ingress (900 GB/s per direction)
    # does not bind at <= 8 links of ~57 GB/s.
    gset = sorted(set(path_gpus))
    conc = conc_rate(torch, gset)
    dram = dram_read_rate(torch)
    terms = {"h2d": {"pcie_sum": R_h2d, "dram_lb": max(dram, conc["h2d"])},
             "d2h": {"pcie_sum": R_d2h, "dram_lb": max(dram, conc["d2h"])}}
    nvl = None
    relay_gpus = [g for g in gset if g != 0]
    if relay_gpus:        # the target's own link plus everything NVLink brings in / takes out
        try:
            nvl = nvlink_rate(torch, 0, relay_gpus)
            terms["h2d"]["ingress"] = pcie[0]["h2d"] + nvl["ingress"]
            terms["d2h"]["ingress"] = pcie[0]["d2h"] + nvl["egress"]
        except Exception as ex:  # noqa: BLE001 - evidence only
            nvl = {"error": f"{type(ex).__name__}: {ex}"}
    Rh, Rd = min(terms["h2d"].values()), min(terms["d2h"].values())
    R_step = nbytes_step / 2 / (Rh * 1e9) + nbytes_step / 2 / (Rd * 1e9)
    path_roof = {"R_h2d_gbps": round(Rh, 2), "R_d2h_gbps": round(Rd, 2),
                 "binding_h2d": min(terms["h2d"], key=terms["h2d"].get),
                 "binding_d2h": min(terms["d2h"], key=terms["d2h"].get),
                 "frac_h2d": round(h2d_gbps / Rh, 4), "frac_d2h": round(d2h_gbps / Rd, 4),
                 "frac_step": round(value / (nbytes_step / R_step / 1e9), 4),
                 "R_conc": {k2: round(v, 2) for k2, v in conc.items()},
                 "cpu_dram_read_gbps": round(dram, 2),
                 "nvlink_gbps": {k2: round(v, 1) for k2, v in nvl.items()} if nvl and "error" not in nvl else nvl,
                 # SURVEY 8(c) bound: a rate above 1.02 x R is a timing bug, not a result
                 "above_roofline_flag": bool(h2d_gbps > 1.02 * Rh or d2h_gbps > 1.02 * Rd),
                 "pcie_solo": {str(g): {k2: round(v, 2) for k2, v in pcie[g].items()} for g in path_gpus},
                 "note": "DRAM term is a lower bound (CPU threads in a VM may not saturate DRAM); when it "
                         "binds, R is a lower bound and the fraction an upper bound"}

    # ---- duplex: request A's fetch overlapping request B's offload (disjoint blocks) on two
    # streams -- PCIe is full duplex; reported beside the sequential headline, not in it
    duplex = None
    if "offload2" in w:
        s2 = torch.cuda.Stream(device=0)
        a = torch.cuda.Event(enable_timing=True)
        b1 = torch.cuda.Event(enable_timing=True)
        b2 = torch.cuda.Event(enable_timing=True)
        best = None
        for _ in range(3):
            torch.cuda.synchronize(0)
            a.record(stream)
            s2.wait_event(a)
            # the cheaper enqueue first: a copy-engine path issues one DMA per block (~5 us of
            # host time each, DESIGN 5.3), a zero-copy launch takes ~1 ms
            mma.memcpy_d2h_segments(*w["offload2"], 0, stream=s2)
            mma.memcpy_h2d_segments(*w["fetch"], 0, stream=stream)
            b1.record(stream)
            b2.record(s2)
            torch.cuda.synchronize(0)
            ms = max(a.elapsed_time(b1), a.elapsed_time(b2))
            best = ms if best is None else min(best, ms)
        duplex = {"gbps": round(2 * w["bytes"] / (best * 1e-3) / 1e9, 2), "ms": round(best, 3),
                  "what": "fetch of request A (H2D) on one stream while request B's disjoint blocks are "
                          "offloaded (D2H) on another; both through the engine"}
        assert mma.get_last_error() == 0

    # ---- pre-enqueued (secondary): the stream is held by a gate kernel while two
    # steps are enqueued, then released -- the data-plane rate without host issue in the way
    preenq = None
    try:
        nst = 2                                       # 4 calls: within the 4 rotating table buffers
        ga = torch.cuda.Event(enable_timing=True)
        gb = torch.cuda.Event(enable_timing=True)
        best = None
        for _ in range(2):
            torch.cuda.synchronize(0)
            with torch.cuda.stream(stream):
                torch.cuda._sleep(int(2.0e9))          # ~1 s at ~2 GHz: longer than the issue
            ga.record(stream)
            t_issue = time.perf_counter()
            for _ in range(nst):
                run_step(mma, w, 0, stream)
            t_issue = time.perf_counter() - t_issue
            gb.record(stream)
            gb.synchronize()
            ms = ga.elapsed_time(gb)
            best = ms if best is None else min(best, ms)
        preenq = {"gbps": round(nst * nbytes_step / (best * 1e-3) / 1e9, 3), "steps": nst,
                  "host_enqueue_ms_per_step": round(t_issue * 1e3 / nst, 3),
                  "what": "stream gated by a sleep kernel while the steps are enqueued; device time after the "
                          "gate. The enqueue time includes blocking once the GPU's command queue is full "
                          "(131,072 per-block copy-engine DMAs do not fit while gated)"}
        assert mma.get_last_error() == 0
    except Exception as ex:  # noqa: BLE001 - evidence only
        preenq = {"error": f"{type(ex).__name__}: {ex}"}

    # ---- one traced step (engine timeline): which GPUs carried the step, and how
    # concurrently (outside the timed region)
    timeline = None
    try:
        Path("gpurun_out").mkdir(exist_ok=True)
        tpath = f"gpurun_out/bench_trace_n{args.gpus}.json"
        mma.trace_begin()
        run_step(mma, w, 0, stream)
        stream.synchronize()
        mma.trace_end(tpath)
        timeline = timeline_summary(tpath)
        if timeline:
            timeline["file"] = tpath
    except Exception as ex:  # noqa: BLE001 - evidence only
        timeline = {"error": str(ex)}

    # ---- hardware check of the chunk -> path assignment: PCIe bytes per path GPU (NVML)
    try:
        pcie_hw = pcie_hw_check(torch, mma, w, stream, path_gpus, plan_choice.get("chosen") == "dynamic")
    except Exception as ex:  # noqa: BLE001 - evidence only
        pcie_hw = {"error": f"{type(ex).__name__}: {ex}"}

    # the dominant kernel against the ceiling of SM-initiated host traffic on this link: the link's
    # raw byte rate (the native copy's rate x its measured protocol overhead) over the kernel's own
    # measured overhead (SM writes / read completions travel as 128-byte TLPs; the copy engine's as
    # 256-byte ones). A second denominator beside the link peak, derived from two counters.
    try:
        if roof and roof["kernel"] in ("zc_copy_kernel", "zc_bulk_kernel") and roof["path"] == 0 and isinstance(pcie_hw, dict):
            rows = pcie_hw.get(roof["direction"]) or []
            kern_ratio = next((r["ratio"] for r in rows if r["gpu"] == roof["device"] and r["ratio"]), None)
            ce_ratio = CE_PCIE_OVERHEAD[roof["direction"]]
            if kern_ratio:
                ceil = roof["peak"] * ce_ratio / kern_ratio
                roof["sm_tlp_ceiling"] = {
                    "gbps": round(ceil, 2), "frac": round(roof["achieved"] / ceil, 4),
                    "kernel_pcie_over_payload": kern_ratio, "copy_engine_pcie_over_payload": ce_ratio,
                    "how": "peak x copy-engine overhead (profiles/r01_probe_nvml.json, native 4 GiB copy) / "
                           "this kernel's overhead (pcie_hw, this run); the two overhead factors come from "
                           "different runs, so the ceiling is good to about +-2%"}
    except (KeyError, TypeError, ZeroDivisionError, StopIteration):
        pass

    # ---- e2e through the public API: wall clock, host issue + copies + sync every step
    run_step(mma, w, 0, stream)                 # one untimed synchronous step first
    stream.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run_step(mma, w, 0, stream)
        stream.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e = {"value": round(nbytes_step / e2e_s / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": w["bytes"], "d2h_bytes_per_step": w["bytes"],
           "how": "wall clock around the Python binding -> C ABI calls, stream synchronized each step"}

    # ---- native baseline on the same buffers: one cudaMemcpyAsync per segment (config 3, the
    # per-block loop of a paged KV cache's swap) or per tensor / transfer, on the user stream
    native = None
    if not args.quick:
        cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = (1 << 64) - 1   # everything native
        mma.init(cfg)
        for _ in range(2):
            run_step(mma, w, 0, stream)
        stream.synchronize()
        nev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        for i in range(args.steps):
            run_step(mma, w, 0, stream, nev[i])
        stream.synchronize()
        nh = statistics.median(nev[i][0].elapsed_time(nev[i][1]) for i in range(args.steps))
        nd = statistics.median(nev[i][1].elapsed_time(nev[i][2]) for i in range(args.steps))
        native = {"h2d_gbps": round(w["bytes"] / nh / 1e6, 2), "d2h_gbps": round(w["bytes"] / nd / 1e6, 2),
                  "step_gbps": round(nbytes_step / (nh + nd) / 1e6, 2),
                  "what": "one cudaMemcpyAsync per 32 KiB segment on the user stream (single PCIe link)"
                  if "fetch" in w else ("one cudaMemcpyAsync per tensor on the user stream (single PCIe link)"
                                        if "wake" in w else "cudaMemcpyAsync on the user stream (single PCIe link)"),
                  "speedup": round(value / (nbytes_step / (nh + nd) / 1e6), 3)}

    # ---- the metric's path-count axis inside one run (GB/s vs k = 1/2/4/8): the
    # same step with the target plus the first k-1 relays, each set tuned as above
    per_k = None
    if k > 1 and not args.quick and multipath_error is None:
        per_k = {}
        saved = (dict(policy), dict(thresholds))     # the line reports the headline run's choices
        for kk in (1, 2, 4, 8):
            if kk >= k:
                continue
            try:
                prepare(list(range(1, kk)))
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(args.steps):
                    run_step(mma, w, 0, stream)
                b.record(stream)
                b.synchronize()
                ms = a.elapsed_time(b) / args.steps
                per_k[str(kk)] = {"value": round(nbytes_step / (ms * 1e-3) / 1e9, 3), "ms_per_step": round(ms, 3)}
            except Exception as ex:  # noqa: BLE001 - evidence only
                per_k[str(kk)] = {"error": f"{type(ex).__name__}: {ex}"}
        per_k[str(k)] = {"value": round(value, 3), "ms_per_step": round(ms_step, 3), "headline": True}
        policy.clear(); policy.update(saved[0])
        thresholds.clear(); thresholds.update(saved[1])

    # ---- CPU baseline: the oracle on the host cores, bounded sample, N=1 only. Two legs
    # (SURVEY 8(d) "Oracle timing alongside"): T = the path set's threads (1 + 2 per relay)
    # and T ~ nproc (a plan over (nproc + 1) // 2 paths), each the median of >= 5 repetitions
    cpu = None
    if not args.quick and dist.world == 1:
        try:
            cpu = cpu_baseline(k)
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "oracle", "sample": f"failed: {ex}"}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": w["desc"], "paths": k, "path_gpus": path_gpus, "target_gpu": 0,
                   "chunk_bytes": int(cfg.chunk_bytes[0]), "claim_bytes": int(cfg.claim_bytes), "hop": {0: "auto", 1: "ce", 2: "zc", 3: "ce_p2p", 4: "push"}[args.hop],
                   "bytes_per_step": nbytes_step,
                   "fallback_bytes": thresholds or fallback_cfg,
                   "fallback_how": "measured break-even (mma_tune_threshold)" if thresholds else "default (2 chunks)", "l2": f"inputs ({w['bytes'] / GiB:.1f} GiB per direction) exceed the 126 MB L2; no flush",
                   "parallelism": f"1 process drives {k} path GPU(s); torchrun ranks>0 idle on gloo",
                   "visible_devices": vis_note, "multipath_error": multipath_error,
                   "virtual_gpus": (ngpu_vis - torch.cuda.device_count()) or None},
        "per_direction": {"h2d_gbps": round(h2d_gbps, 2), "d2h_gbps": round(d2h_gbps, 2),
                          "h2d_ms": round(h2d_ms, 3), "d2h_ms": round(d2h_ms, 3)},
        "path_roofline": path_roof,
        "roofline": roof,
        "native": native,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "timeline": timeline,
        "duplex": duplex,
        "pcie_hw": pcie_hw,
        "preenqueued": preenq,
        "gpu_launches": int(st["kernels"]),
        "kernel_kinds": kinds,
        "clocks": clk,
        "host_cpu": host_cpu,
        "verify": verify,
        "plan": plan_choice,
        "mode_policy": policy or None,
        "per_path_count": per_k,
        "numa": numa_info(torch, sorted(set(path_gpus))),
        "topology": topology,
        "modes": {d: [{"gpu": pi["gpu"], "mode": {0: "auto", 1: "ce", 2: "zc", 3: "ce_p2p", 4: "push"}.get(
            pi["seg_mode"] if ("fetch" in w and pi["seg_mode"] >= 0) else pi["mode"], "?"),
            "mbps": pi["seg_mbps"] if ("fetch" in w and pi["seg_mbps"]) else pi["mbps"]} for pi in v]
            for d, v in tuned.items()},
        "calibration": {"per_path_mbps": calib, "rounds": int(cfg.calib_rounds),
                        "what": "solo = the path alone in its chosen mode; conc = with every path of the set "
                                "active (0: single path, not refined)"},
        "engine": {"issue_us_per_call": round((st["issue_us"] - st["wait_us"]) / max(1, st["calls"]), 1),
                   "enqueue_cpu_percent": round(100 * (st["issue_us"] - st["wait_us"]) / max(1e-9, 1e3 * ms_total), 1),
                   "blocked_us_per_call": round(st["wait_us"] / max(1, st["calls"]), 1),
                   "relay_bytes": int(st["relay_bytes"]), "fallbacks": int(st["fallbacks"]),
                   "single_path_calls": int(st["single_path_calls"]),
                   "validate_us_per_call": round(st["validate_us"] / max(1, st["calls"]), 1),
                   "numa_local_of_known_bytes": [int(st["numa_local_bytes"][0]), int(st["numa_known_bytes"][0]),
                                                 int(st["numa_local_bytes"][1]), int(st["numa_known_bytes"][1])]},
        "paper_context": "245 GB/s = 4.62x one 53 GB/s PCIe link, 8x H20 (P:737); context only",
    }
    print(json.dumps(line), flush=True)
    dist.close()


if __name__ == "__main__":
    try:
        main()
    except Exception as ex:  # noqa: BLE001 - a failed run still leaves one parseable line
        if int(os.environ.get("RANK", 0)) == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": "GB/s", "error": f"{type(ex).__name__}: {ex}"}),
                  flush=True)
        raise
