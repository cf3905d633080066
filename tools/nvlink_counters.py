"""NVLink byte counters through NVML field values (no nsys / DCGM in this
image, and ncu cannot replay a kernel whose peers run in other processes).

  LinkCounters(device).read() -> {"tx": bytes, "rx": bytes, "links": n, "field": name}

Tries, in order, the per-link data counters NVML exposes on Blackwell:
NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES (202 / 204, bytes) and
NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX (138 / 139, KiB), each summed
over the GPU's links (scopeId = link). `python tools/nvlink_counters.py`
probes every field around a 1 GiB peer copy between GPU 0 and GPU 1.
"""
from __future__ import annotations

import sys

FIELDS = [("count_bytes", 202, 204, 1), ("throughput_data_kib", 138, 139, 1024),
          ("throughput_raw_kib", 140, 141, 1024)]


class LinkCounters:
    def __init__(self, device: int):
        import pynvml as nv
        nv.nvmlInit()
        self.nv = nv
        self.h = nv.nvmlDeviceGetHandleByIndex(device)
        self.links = []
        for link in range(18):
            try:
                if nv.nvmlDeviceGetNvLinkState(self.h, link) == nv.NVML_FEATURE_ENABLED:
                    self.links.append(link)
            except Exception:
                break
        self.field = None
        for name, tx, rx, scale in FIELDS:
            vals = self._sample(tx, rx, scale)
            if vals is not None:
                self.field = (name, tx, rx, scale)
                break

    def _sample(self, tx_id: int, rx_id: int, scale: int):
        nv = self.nv
        if not self.links:
            return None
        req = []
        for link in self.links:
            req.append((tx_id, link))
            req.append((rx_id, link))
        try:
            out = nv.nvmlDeviceGetFieldValues(self.h, req)
        except Exception:
            return None
        tx = rx = 0
        for k, v in enumerate(out):
            if v.nvmlReturn != 0:
                return None
            val = v.value.ullVal if v.valueType in (1, 3, 5) else v.value.uiVal
            if v.valueType == 0:
                val = v.value.dVal
            if k % 2 == 0:
                tx += val
            else:
                rx += val
        return tx * scale, rx * scale

    def read(self) -> dict | None:
        if self.field is None:
            return None
        name, tx, rx, scale = self.field
        vals = self._sample(tx, rx, scale)
        if vals is None:
            return None
        return {"tx": vals[0], "rx": vals[1], "links": len(self.links), "field": name}


def probe():
    import torch
    import pynvml as nv
    nv.nvmlInit()
    n = torch.cuda.device_count()
    print("devices", n)
    h = nv.nvmlDeviceGetHandleByIndex(0)
    links = []
    for link in range(18):
        try:
            st = nv.nvmlDeviceGetNvLinkState(h, link)
            links.append((link, st))
        except Exception as e:
            links.append((link, f"err {e}"))
    print("links", links)
    ids = [138, 139, 140, 141, 201, 202, 203, 204]

    def snap():
        res = {}
        for fid in ids:
            row = []
            for link in (0, 1, 0xFFFFFFFF):
                try:
                    v = nv.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                    row.append((v.nvmlReturn, v.valueType, v.value.ullVal))
                except Exception as e:
                    row.append(str(e)[:40])
            res[fid] = row
        return res

    a = snap()
    if n >= 2:
        x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
        y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
        for _ in range(4):
            y.copy_(x)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
    b = snap()
    for fid in ids:
        print(fid, "before", a[fid], "after", b[fid])
    c = LinkCounters(0)
    print("LinkCounters field", c.field, "links", c.links, c.read())


if __name__ == "__main__":
    sys.exit(probe())
