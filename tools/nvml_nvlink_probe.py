"""Which NVML NVLink counters move during a P2P copy (GPU0 -> GPU1)? Prints per field id the
summed per-link value before/after a 1 GiB peer copy, and the return codes."""
import pynvml
import torch

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
links = []
for l in range(18):
    try:
        if pynvml.nvmlDeviceGetNvLinkState(h, l):
            links.append(l)
    except Exception as e:  # noqa: BLE001
        pass
print("links up", links)
FIELDS = {138: "THROUGHPUT_DATA_TX", 139: "THROUGHPUT_DATA_RX", 140: "THROUGHPUT_RAW_TX", 141: "THROUGHPUT_RAW_RX",
          201: "COUNT_XMIT_PACKETS", 202: "COUNT_XMIT_BYTES", 203: "COUNT_RCV_PACKETS", 204: "COUNT_RCV_BYTES"}


def read():
    out = {}
    for f in FIELDS:
        for scope in (links, [0xFFFFFFFF]):
            ids = [(f, l) for l in scope]
            try:
                vals = pynvml.nvmlDeviceGetFieldValues(h, ids)
            except Exception as e:  # noqa: BLE001
                out[(f, len(scope))] = f"err {e}"
                continue
            rets = {v.nvmlReturn for v in vals}
            out[(f, len(scope))] = (sum(int(v.value.ullVal) for v in vals if v.nvmlReturn == 0), sorted(rets))
    return out


a = torch.empty(1 << 28, dtype=torch.float32, device="cuda:0").fill_(1)
b = torch.empty(1 << 28, dtype=torch.float32, device="cuda:1")
torch.cuda.synchronize()
r0 = read()
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize()
r1 = read()
for k in r0:
    print(FIELDS[k[0]], "links" if k[1] > 1 else "all", r0[k], r1[k])
print("copied bytes", 4 * 4 * (1 << 28))
