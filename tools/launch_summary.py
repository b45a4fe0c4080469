"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X.csv python bench.py ...`): total device time, the share of this
library's kernels (namespace fsdp::), and the top kernels by share.

    python tools/launch_summary.py launches.csv [steps_captured] > summary.txt
"""
import csv
import sys
from collections import defaultdict


# kernels defined in paper_2304_11277_b200/csrc (ncu prints them with or
# without the fsdp:: namespace depending on its name-base setting)
OURS = ("adam_kernel", "adam_tma_kernel", "allgather_kernel", "allgather_ll_kernel", "allgather_nvls_kernel",
        "allreduce_kernel", "ar_epilogue_kernel", "cast_kernel", "ce_reduce_kernel", "coll_enter_kernel",
        "coll_exit_kernel", "coll_signal_kernel", "coll_signal_exit_kernel", "fold_error_kernel", "coll_signal_slot_kernel", "coll_wait_slot_kernel",
        "flatten_kernel", "reduce_scatter_kernel", "reduce_scatter_ll_kernel", "reduce_scatter_pull_kernel",
        "reduce_scatter_tma_kernel", "scalar_allreduce_kernel", "sgd_kernel", "unflatten_kernel",
        "unscale_kernel", "shard_copy_kernel")


def is_ours(name: str) -> bool:
    if "fsdp::" in name:
        return True
    base = name.split("(")[0].split("<")[0].split()[-1] if name.strip() else ""
    return base in OURS


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        tot[r[ki]] += us
        cnt[r[ki]] += 1
    total = sum(tot.values())
    ours = sum(v for k, v in tot.items() if is_ours(k))
    n = sum(cnt.values())
    print(f"total {total / 1e3:.1f} ms over {n} launches"
          + (f" = {total / 1e3 / steps:.1f} ms/step ({steps} steps captured)" if steps else ""))
    print(f"fsdp_b200 kernels: {100 * ours / total:.2f}% of device time")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:40]:
        print(f"{100 * v / total:6.2f}% {cnt[k]:6d} {v / cnt[k]:10.1f}us {k[:110]}")


if __name__ == "__main__":
    main()
