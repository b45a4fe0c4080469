"""Per-category device-memory ledger of one rank (the reference's
`MemoryLedger`, memsim.py:113-185, kept on the real runtime).

The categories are the reference's (memsim.py:13-14).  What each one holds
on the B200 runtime:

  sharded_params    fp32 master shards, plus the bf16 copy Adam's epilogue
                    writes (the all-gather source) under mixed precision
  unsharded_params  gathered units resident in symmetric slots, compute dtype
                    (booked at `_issue_unshard`, released at `reshard`,
                    engine.py:654-664, :739-749)
  grads             fp32 reduced-gradient shards (resident arena), the
                    unsharded payload of a unit between write-back and its
                    reduction (engine.py:530), the no_comm fp32 accumulator
                    (engine.py:761)
  activations       torch-allocator bytes above the resident state, sampled
                    after every unit's forward (engine.py:489)
  optimizer_state   Adam exp_avg + exp_avg_sq shards (engine.py:347)

Slots and gradient slots live in the communicator's symmetric pool, which is
allocated once outside torch's caching allocator; the ledger books what is
*in use*, exactly as the reference books its simulated blocks, so the
reference's closed-form peak (`peak_param_bytes`, flatparam.py:198-235) can be
checked against a real run (`verify --serialized`).
"""
from __future__ import annotations

CATEGORIES = ("sharded_params", "unsharded_params", "grads", "activations", "optimizer_state")


class MemoryLedger:
    def __init__(self) -> None:
        self.current_bytes = dict.fromkeys(CATEGORIES, 0)
        self.current_elements = dict.fromkeys(CATEGORIES, 0)
        self.peak_bytes = dict.fromkeys(CATEGORIES, 0)
        self.peak_elements = dict.fromkeys(CATEGORIES, 0)
        self.peak_total_bytes = 0
        self.peak_param_bytes = 0
        self.peak_param_elements = 0

    def _after(self, cat: str) -> None:
        cb, ce = self.current_bytes, self.current_elements
        self.peak_bytes[cat] = max(self.peak_bytes[cat], cb[cat])
        self.peak_elements[cat] = max(self.peak_elements[cat], ce[cat])
        self.peak_total_bytes = max(self.peak_total_bytes, sum(cb.values()))
        self.peak_param_bytes = max(self.peak_param_bytes, cb["sharded_params"] + cb["unsharded_params"])
        self.peak_param_elements = max(self.peak_param_elements,
                                       ce["sharded_params"] + ce["unsharded_params"])

    def alloc(self, cat: str, nbytes: int, elements: int) -> None:
        self.current_bytes[cat] += int(nbytes)
        self.current_elements[cat] += int(elements)
        self._after(cat)

    def free(self, cat: str, nbytes: int, elements: int) -> None:
        self.current_bytes[cat] -= int(nbytes)
        self.current_elements[cat] -= int(elements)
        if self.current_bytes[cat] < 0:
            raise AssertionError(f"negative {cat} bytes")
        self._after(cat)

    def set_level(self, cat: str, nbytes: int) -> None:
        """Sampled category (activations): current level, peak kept."""
        self.current_bytes[cat] = max(0, int(nbytes))
        self._after(cat)

    def reset_peaks(self) -> dict:
        """Restart peak tracking from the current residency (separates the
        initialisation phase from training, engine.py:355); returns the old peaks."""
        old = self.snapshot()
        cb, ce = self.current_bytes, self.current_elements
        self.peak_bytes = dict(cb)
        self.peak_elements = dict(ce)
        self.peak_total_bytes = sum(cb.values())
        self.peak_param_bytes = cb["sharded_params"] + cb["unsharded_params"]
        self.peak_param_elements = ce["sharded_params"] + ce["unsharded_params"]
        return old

    def snapshot(self) -> dict:
        return {"current_bytes": dict(self.current_bytes), "peak_bytes": dict(self.peak_bytes),
                "peak_elements": dict(self.peak_elements), "peak_total_bytes": self.peak_total_bytes,
                "peak_param_bytes": self.peak_param_bytes, "peak_param_elements": self.peak_param_elements}


def peak_param_bytes(psis, shard_numels, shard_factor: int, k_full: int = 4, k_low: int | None = 2,
                     low_copy: bool = True, variant: str = "serialized", nested_root: bool = False) -> int:
    """flatparam.py:198-235 (peak_param_memory) for this runtime's layout:
    resident shards in full precision (k_full per element, plus the k_low
    bf16 copy when `low_copy`), plus the gathered units in k_low (serialized:
    the largest one; two_inflight: the two largest).  F = 1 gathers nothing.

    nested_root: unit 0 is the wrapper's root, whose forward encloses every
    other unit (torch-FSDP nesting; the reference's units are sequential), so
    it stays gathered while each child is: serialized peak = root + the
    largest child (two_inflight: root + the two largest children)."""
    shards = sum(shard_numels)
    res = shards * k_full + (shards * k_low if (low_copy and k_low) else 0)
    if shard_factor == 1 or not psis:
        return res
    k = k_low if k_low else k_full
    if nested_root:
        kids = sorted(psis[1:], reverse=True)
        return res + (psis[0] + sum(kids[:1] if variant == "serialized" else kids[:2])) * k
    largest = sorted(psis, reverse=True)
    gathered = largest[:1] if variant == "serialized" else largest[:2]
    return res + sum(gathered) * k
