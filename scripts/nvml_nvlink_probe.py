"""Which NVML NVLink byte counters move on this box: copies 1 GiB GPU0 -> GPU1
peer-to-peer and prints every candidate field (per link and aggregate)."""
import pynvml as N
import torch

N.nvmlInit()
hd = [N.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
FIELDS = {"THROUGHPUT_DATA_TX": 138, "THROUGHPUT_DATA_RX": 139, "THROUGHPUT_RAW_TX": 140, "THROUGHPUT_RAW_RX": 141,
          "COUNT_XMIT_BYTES": 202, "COUNT_RCV_BYTES": 204}


def read(h):
    out = {}
    for name, fid in FIELDS.items():
        for scope in list(range(18)) + [0xFFFFFFFF]:
            try:
                v = N.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            except Exception as e:  # noqa: BLE001
                out[(name, scope)] = f"exc {e}"
                continue
            if v.nvmlReturn != 0:
                out[(name, scope)] = f"ret {v.nvmlReturn}"
                continue
            out[(name, scope)] = (v.valueType, v.value.ullVal, v.value.ulVal, v.value.uiVal)
    return out


for i, h in enumerate(hd):
    st = []
    for l in range(18):
        try:
            st.append(N.nvmlDeviceGetNvLinkState(h, l))
        except Exception as e:  # noqa: BLE001
            st.append(str(e)[:20])
    print("gpu", i, "link states", st)
b0 = read(hd[0])
a = torch.empty(1 << 28, dtype=torch.float32, device="cuda:0")
b = torch.empty(1 << 28, dtype=torch.float32, device="cuda:1")
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
b1 = read(hd[0])
for k in b0:
    if b0[k] != b1[k]:
        print("CHANGED", k, b0[k], "->", b1[k])
print("sample", {k: b1[k] for k in list(b1)[:6]})
