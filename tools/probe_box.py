"""Probe the GPU box: NVLink multicast (NVLS) support and NVML NVLink
throughput counters, with a peer copy to check that the counters move.

Writes one JSON line to stdout. Used to decide whether a multicast
all-gather is possible on this pool's boxes.
"""
import json
import time

import torch
from cuda.bindings import driver as d
import pynvml


def main():
    out = {}
    d.cuInit(0)
    n = torch.cuda.device_count()
    out["n_gpus"] = n
    for i in range(n):
        err, dev = d.cuDeviceGet(i)
        a = d.CUdevice_attribute
        out[f"gpu{i}"] = {
            "multicast": d.cuDeviceGetAttribute(a.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)[1],
            "vmm": d.cuDeviceGetAttribute(a.CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev)[1],
            "fabric_handle": d.cuDeviceGetAttribute(a.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)[1],
            "posix_fd_handle": d.cuDeviceGetAttribute(a.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev)[1],
        }
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    fields = [pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
              pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX, pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX]

    def read():
        vals = pynvml.nvmlDeviceGetFieldValues(h, fields)
        res = []
        for v in vals:
            if v.nvmlReturn != 0:
                res.append(None)
            else:
                res.append(int(v.value.ullVal))
        return res

    out["nvml_before"] = read()
    if n >= 2:
        a_ = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
        b_ = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
        torch.cuda.synchronize(0)
        r0 = read()
        t = time.time()
        for _ in range(8):
            b_.copy_(a_)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        time.sleep(0.5)
        r1 = read()
        out["copy_bytes"] = 8 << 30
        out["nvml_delta"] = [None if x is None or y is None else y - x for x, y in zip(r0, r1)]
        out["copy_s"] = time.time() - t
    try:
        nl = []
        for link in range(18):
            try:
                nl.append(pynvml.nvmlDeviceGetNvLinkState(h, link))
            except pynvml.NVMLError as e:
                nl.append(str(e))
        out["nvlink_state"] = nl
    except Exception as e:  # noqa: BLE001
        out["nvlink_state"] = str(e)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
