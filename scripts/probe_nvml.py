"""Probe: NVML's cumulative PCIe byte counters on this B200 (SURVEY 8(d) "hardware-level
check of the chunk-to-path assignment"): width (they wrap), update period, and the bytes
they count around a 4 GiB H2D and D2H copy, sampled from a thread every ~1 ms."""
import json
import threading
import time

import pynvml as N
import torch

N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
F = [N.NVML_FI_DEV_PCIE_COUNT_RX_BYTES, N.NVML_FI_DEV_PCIE_COUNT_TX_BYTES]


def read():
    v = N.nvmlDeviceGetFieldValues(h, F)
    return time.perf_counter(), int(v[0].value.ullVal), int(v[1].value.ullVal)


def sample(stop, out):
    while not stop.is_set():
        out.append(read())
        time.sleep(0.001)


B = 4 << 30
src = torch.empty(B, dtype=torch.uint8).pin_memory()
dst = torch.empty(B, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200):
    read()
res = {"read_us": (time.perf_counter() - t) / 200 * 1e6}
for name, fn in [("h2d", lambda: dst.copy_(src, non_blocking=True)), ("d2h", lambda: src.copy_(dst, non_blocking=True))]:
    s, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, s))
    th.start()
    time.sleep(0.05)
    fn()
    torch.cuda.synchronize()
    time.sleep(0.3)
    stop.set()
    th.join()
    col = 1 if name == "h2d" else 2
    changes = [(round((b[0] - s[0][0]) * 1e3, 2), (b[col] - a[col]) % (1 << 32)) for a, b in zip(s, s[1:]) if b[col] != a[col]]
    tot = sum(d for _, d in changes)
    res[name] = {"samples": len(s), "changes": len(changes), "first_changes_ms_bytes": changes[:12],
                 "max_raw": max(x[col] for x in s), "unwrapped_total": tot, "ratio_to_payload": tot / B}
print(json.dumps(res, indent=1))
