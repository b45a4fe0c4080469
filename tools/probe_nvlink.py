"""Which NVML NVLink byte counters move on this box?  Reads fields 138-141
(throughput KiB) and 202/204 (xmit/rcv bytes), device-wide and per link
(scopeId = link), around an 8 GiB GPU0 -> GPU1 copy."""
import json

import pynvml
import torch

FIELDS = {"tput_data_tx": 138, "tput_data_rx": 139, "tput_raw_tx": 140, "tput_raw_rx": 141,
          "xmit_bytes": 202, "rcv_bytes": 204}


def read(h):
    out = {}
    for name, fid in FIELDS.items():
        for scope in [None] + list(range(18)):
            req = [fid if scope is None else (fid, scope)]
            try:
                v = pynvml.nvmlDeviceGetFieldValues(h, req)[0]
            except pynvml.NVMLError as e:
                out[f"{name}@{scope}"] = f"err {e}"
                continue
            out[f"{name}@{scope}"] = int(v.value.ullVal) if v.nvmlReturn == 0 else f"ret {v.nvmlReturn}"
    return out


def main():
    pynvml.nvmlInit()
    h0 = pynvml.nvmlDeviceGetHandleByIndex(0)
    a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
    torch.cuda.synchronize(0)
    r0 = read(h0)
    for _ in range(8):
        b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    import time
    time.sleep(1.0)
    r1 = read(h0)
    delta = {}
    for k in r0:
        if isinstance(r0[k], int) and isinstance(r1[k], int):
            delta[k] = r1[k] - r0[k]
        else:
            delta[k] = r1[k]
    agg = {}
    for name in FIELDS:
        per = [delta.get(f"{name}@{l}") for l in range(18)]
        agg[name] = {"device": delta.get(f"{name}@None"),
                     "sum_links": sum(x for x in per if isinstance(x, int)) if any(isinstance(x, int) for x in per) else per[0]}
    print(json.dumps({"copied_bytes": 8 << 30, "agg": agg}))


if __name__ == "__main__":
    main()
