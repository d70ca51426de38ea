#!/usr/bin/env python3
"""Condense the ncu reports of scripts/profile_round.sh (gpurun_out/*.ncu-rep, read here with
`ncu -i`) into profiles/: per-kernel raw/details CSVs, the launch list, and
profiles/ncu_summary.json (bench.py reads `traffic` from its dram_bytes_per_launch).

Algorithmic bytes per launch: zero-copy gather/scatter moves the config-3
payload once (4 GiB); HBM traffic should be 1 B per payload byte (write for H2D, read for
D2H). The relay kernels read the staging slot and write the destination: 2 B per payload
byte of HBM traffic on one GPU (loopback), the payload being 7 rings x 256 MiB."""
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"

KV_BYTES = 131072 * 32768
RELAY_BYTES = 7 * 32 * (8 << 20)


def ncu_csv(rep, page):
    r = subprocess.run(["ncu", "-i", str(rep), "--page", page, "--csv"], capture_output=True, text=True, check=True)
    return r.stdout


def raw_rows(rep):
    rows = list(csv.reader(io.StringIO(ncu_csv(rep, "raw"))))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = {}
        for k, u, v in zip(hdr, units, row):
            d[k] = (v, u)
        out.append(d)
    return out


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3, "nsecond": 1e-6}


def val(d, k, to="byte"):
    if k not in d:
        return None
    v, u = d[k]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * SCALE.get(u, 1.0)


def kernel_entry(d, what, algo, source):
    t_ms = val(d, "gpu__time_duration.sum")
    rd, wr = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
    e = {"what": what, "source": source, "gpu_time_ms": round(t_ms, 3) if t_ms else None,
         "grid": d.get("launch__grid_size", ("?",))[0],
         "regs_per_thread": d.get("launch__registers_per_thread", ("?",))[0],
         "dram_bytes_read": int(rd) if rd is not None else None,
         "dram_bytes_write": int(wr) if wr is not None else None,
         "algorithmic_bytes_per_launch": algo}
    if rd is not None and wr is not None:
        e["dram_bytes_per_launch"] = int(rd + wr)
    for k in ("pcie__read_bytes.sum", "pcie__write_bytes.sum"):
        if val(d, k) is not None:
            e[k.split(".")[0]] = int(val(d, k))
    return e


def zc_name(d):
    """zc_copy_kernel (vector form) or zc_bulk_kernel (cp.async.bulk form) from the row's kernel name"""
    import re
    m = re.search(r"(zc_\w+?_kernel)", d.get("Kernel Name", ("",))[0])
    return m.group(1) if m else "zc_copy_kernel"


def main():
    PROF.mkdir(exist_ok=True)
    summary = {"source": f"scripts/profile_round.sh on 1 x B200 (ncu --clock-control none), round {TAG}",
               "kernels": {}, "dram_bytes_per_launch": {}}
    h2d = OUT / "prof_zc_h2d.ncu-rep"
    if h2d.exists():
        (PROF / f"{TAG}_ncu_zc_h2d_details.csv").write_text(ncu_csv(h2d, "details"))
        d = raw_rows(h2d)[0]
        e = kernel_entry(d, "SM zero-copy gather (" + zc_name(d) + ") of the config-3 KV fetch (131072 x 32 KiB host segments -> "
                            "paged device cache), one launch", KV_BYTES, f"profiles/{TAG}_ncu_zc_h2d_details.csv")
        e["note"] = ("HBM traffic ~= algorithmic (each payload byte written once; host reads cross PCIe, not "
                     "DRAM): no re-reads")
        summary["kernels"][f"{zc_name(d)}/h2d"] = e
        summary["dram_bytes_per_launch"]["h2d"] = e.get("dram_bytes_per_launch")
    d2h = OUT / "prof_zc_d2h.ncu-rep"
    if d2h.exists():
        (PROF / f"{TAG}_ncu_zc_d2h_metrics.csv").write_text(ncu_csv(d2h, "raw"))
        d = raw_rows(d2h)[0]
        e = kernel_entry(d, "SM zero-copy scatter (" + zc_name(d) + ") of the config-3 KV offload (paged device cache -> 131072 x "
                            "32 KiB host slots), one launch; application replay (host-writing kernels return nan "
                            "under kernel replay)", KV_BYTES, f"profiles/{TAG}_ncu_zc_d2h_metrics.csv")
        if e.get("pcie__write_bytes"):
            e["pcie_write_over_payload"] = round(e["pcie__write_bytes"] / KV_BYTES, 4)
        summary["kernels"][f"{zc_name(d)}/d2h"] = e
        summary["dram_bytes_per_launch"]["d2h"] = e.get("dram_bytes_per_launch")
    rel = OUT / "prof_relay.ncu-rep"
    if rel.exists():
        (PROF / f"{TAG}_ncu_relay_details.csv").write_text(ncu_csv(rel, "details"))
        for d in raw_rows(rel):
            name = d["Kernel Name"][0].split("(")[0].split("::")[-1]
            e = kernel_entry(d, f"{name} alone (scripts/probe/probe_relay ncu): 7 rings x 8 CTAs, 8 MiB chunks, "
                                "hop 1 complete, slots in local HBM (loopback)", RELAY_BYTES,
                             f"profiles/{TAG}_ncu_relay_details.csv")
            e["algorithmic_hbm_bytes_per_launch"] = 2 * RELAY_BYTES
            if e["gpu_time_ms"]:
                e["payload_gbps"] = round(RELAY_BYTES / (e["gpu_time_ms"] * 1e-3) / 1e9, 1)
            summary["kernels"][name] = e
    rel = OUT / "prof_relay_seg.ncu-rep"
    if rel.exists():
        (PROF / f"{TAG}_ncu_relay_seg_details.csv").write_text(ncu_csv(rel, "details"))
        for d in raw_rows(rel):
            name = d["Kernel Name"][0].split("(")[0].split("::")[-1] + "/scattered"
            e = kernel_entry(d, f"{name} alone, C3 scattered form: v = 32 KiB segments at permuted blocks, "
                                "7 rings x 8 CTAs, hop 1 complete, local HBM", RELAY_BYTES,
                             f"profiles/{TAG}_ncu_relay_seg_details.csv")
            e["algorithmic_hbm_bytes_per_launch"] = 2 * RELAY_BYTES
            if e["gpu_time_ms"]:
                e["payload_gbps"] = round(RELAY_BYTES / (e["gpu_time_ms"] * 1e-3) / 1e9, 1)
            summary["kernels"][name] = e
    for rel, sfx in ((OUT / "prof_relay_proto.ncu-rep", ""), (OUT / "prof_relay_proto_pull.ncu-rep", "_pull")):
        if not rel.exists():
            continue
        (PROF / f"{TAG}_ncu_relay_protocol{sfx}_details.csv").write_text(ncu_csv(rel, "details"))
        (PROF / f"{TAG}_ncu_relay_protocol{sfx}_raw.csv").write_text(ncu_csv(rel, "raw"))
        for k, d in enumerate(raw_rows(rel)):
            name = d["Kernel Name"][0].split("(")[0].split("::")[-1]
            grid = int(str(d.get("launch__grid_size", ("0",))[0]).replace(",", "") or 0)
            # one wave: 3 rings x S = 4 chunks x 8 MiB (loopback form)
            algo = 3 * 4 * (8 << 20)
            e = kernel_entry(d, f"{name} in the engine's protocol (scripts/ncu_relay_protocol.py): one wave of "
                                "3 rings x 4 chunks x 8 MiB, launched by mma_memcpy_* after (H2D) / before (D2H) "
                                "the wave's hops; ncu serialises, so the wave's hop 1 is complete", algo,
                             f"profiles/{TAG}_ncu_relay_protocol{sfx}_details.csv")
            e["algorithmic_hbm_bytes_per_launch"] = 2 * algo
            for m in ("nvlrx__bytes.sum", "nvltx__bytes.sum"):
                if val(d, m) is not None:
                    e[m.split(".")[0]] = int(val(d, m))
            if e["gpu_time_ms"]:
                e["payload_gbps"] = round(algo / (e["gpu_time_ms"] * 1e-3) / 1e9, 1)
            e["launch"] = k
            summary["kernels"][f"{name}/protocol/{k}"] = e
    lst = OUT / "launches_bench.csv"
    if lst.exists():
        shutil.copy(lst, PROF / f"{TAG}_launches_bench.csv")
    (PROF / "ncu_summary.json").write_text(json.dumps(summary, indent=2) + "\n")
    print(json.dumps(summary, indent=2))


if __name__ == "__main__":
    main()
