"""Device communicator: symmetric CUDA-IPC pool + SM-driven collectives.

`DeviceComm` owns one `fsdp_comm_t` (include/fsdp_b200.h).  It is created
either
  * for real (`DeviceComm.create`): one process per GPU; IPC handles of every
    rank's pool are exchanged once with torch.distributed (plumbing only),
  * or emulated (`DeviceComm.create_emulated`): all W ranks' pools on the
    current GPU, each collective one cooperative launch over every rank's
    data — used to test the cross-rank protocol on a single B200.

Pool regions are handed out by a deterministic bump allocator, so every rank
obtains the same offsets for the same sequence of `alloc` calls (symmetric
addressing: a collective names a destination by offset only).

`DeviceFabric` is the shardsim-shaped functional front end
(collectives.py:183-203): all_gather / reduce_scatter / all_reduce on 1-D
tensors with the reference's entry contract (CollectiveError on a non-member
rank, a non-1-D buffer, or a length not divisible by the group).
"""
from __future__ import annotations

import ctypes as C
import os
import socket
from typing import Sequence

import torch

from . import _lib
from ._lib import check, lib
from .plan import CollectiveError, DeadlockError, group_desc_of

_DT = {torch.float32: _lib.F32, torch.bfloat16: _lib.BF16}
_ES = {torch.float32: 4, torch.bfloat16: 2}


def dtype_code(dt: torch.dtype) -> int:
    try:
        return _DT[dt]
    except KeyError:
        raise CollectiveError(f"unsupported dtype {dt}; fp32 and bf16 are supported") from None


class _CudaBuffer:
    """__cuda_array_interface__ wrapper: a torch view of raw device memory."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def raw_tensor(ptr: int, nbytes: int, device: torch.device) -> torch.Tensor:
    return torch.as_tensor(_CudaBuffer(ptr, nbytes), device=device)


def stream_ptr(stream: torch.cuda.Stream | None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _fd_passing_ok() -> bool:
    return hasattr(socket, "send_fds") and hasattr(socket, "AF_UNIX")


def _handle_bytes(fd: int) -> bytes:
    return int(fd).to_bytes(4, "little", signed=True) + bytes(_lib.SHAREABLE_BYTES - 4)


class _FdBox:
    """File-descriptor exchange between the ranks' processes (SCM_RIGHTS over
    abstract-namespace Unix sockets): the POSIX-fd shareable handles of
    cuMemExportToShareableHandle are process-local numbers."""

    def __init__(self, token: str, rank: int):
        self.token, self.rank = token, rank
        self.sock = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        self.sock.bind(self._addr(rank))
        self.sock.listen(64)
        self.sock.settimeout(120.0)

    def _addr(self, r: int) -> str:
        return f"\0fsdp-b200-{self.token}-{r}"

    def exchange(self, sends: dict, n_recv: int, tag: int) -> dict:
        for peer, fd in sends.items():
            c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            c.settimeout(120.0)
            c.connect(self._addr(peer))
            socket.send_fds(c, [bytes([tag]) + self.rank.to_bytes(4, "little")], [fd])
            c.close()
        got = {}
        while len(got) < n_recv:
            conn, _ = self.sock.accept()
            msg, fds, _, _ = socket.recv_fds(conn, 16, 1)
            conn.close()
            if not fds or len(msg) < 5 or msg[0] != tag:
                for f in fds:
                    os.close(f)
                raise RuntimeError("unexpected fd message")
            got[int.from_bytes(msg[1:5], "little")] = fds[0]
        return got

    def close(self) -> None:
        self.sock.close()


class DeviceComm:
    def __init__(self, handle: int, rank: int, world: int, emulated: bool, device: torch.device):
        self._h = C.c_void_p(handle)
        self.rank, self.world, self.emulated = rank, world, emulated
        self.device = device
        self.pool_bytes = int(lib.fsdp_comm_pool_bytes(self._h))
        self.reserved = int(lib.fsdp_comm_reserved_bytes())
        self._cursor = self.reserved
        nviews = world if emulated else 1
        self._pools = []
        for e in range(nviews):
            r = e if emulated else rank
            ptr = lib.fsdp_comm_pool_ptr(self._h, r)
            self._pools.append(raw_tensor(ptr, self.pool_bytes, device))
        self.closed = False

    # ------------------------------------------------------------ creation --
    @classmethod
    def create(cls, pool_bytes: int, max_ctas: int = 32, group=None,
               nvls_group: int | None = None) -> "DeviceComm":
        """Real communicator over the ranks of `group`.

        nvls_group=F (F > 1, F | world) first tries an exportable VMM pool
        bound to the NVLink SHARP multicast object of each consecutive group
        of F ranks (`all_gather_nvls`); every rank falls back together to the
        cudaMalloc + CUDA-IPC pool if any step fails anywhere."""
        import torch.distributed as dist
        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        if nvls_group and nvls_group > 1 and world % nvls_group == 0:
            comm = cls._create_vmm(pool_bytes, max_ctas, group, nvls_group, rank, world, dev)
            if comm is not None:
                return comm
        h = C.c_void_p()
        check(lib.fsdp_comm_create(rank, world, pool_bytes, max_ctas, C.byref(h)), "comm_create")
        buf = (C.c_char * _lib.IPC_HANDLE_BYTES)()
        check(lib.fsdp_comm_ipc_handle(h, buf), "comm_ipc_handle")
        mine = bytes(buf)
        handles: list = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        allh = b"".join(handles)
        check(lib.fsdp_comm_open_peers(h, allh), "comm_open_peers")
        torch.cuda.synchronize()
        dist.barrier(group=group)          # every pool's flags are zeroed before use
        return cls(h.value, rank, world, False, dev)

    @classmethod
    def _create_vmm(cls, pool_bytes, max_ctas, group, F, rank, world, dev):
        """VMM pool + NVLS multicast; None on every rank if any rank fails.

        Every phase runs locally under try/except and ends in an all-gather
        of (ok, message), so all ranks leave together: a local failure never
        leaves a peer waiting in a different collective."""
        import torch.distributed as dist

        def agree(ok: bool, what: str) -> tuple[bool, str]:
            st: list = [None] * world
            dist.all_gather_object(st, (ok, what), group=group)
            bad = [w for o, w in st if not o]
            return (not bad), (bad[0] if bad else "")

        def attempt(fn) -> tuple[bool, str]:
            try:
                fn()
                return agree(True, "")
            except Exception as exc:  # noqa: BLE001 — reported to every rank
                return agree(False, f"rank {rank}: {exc}")

        h = C.c_void_p()
        state = {"own_fd": -1, "mc_fd": -1, "box": None, "created": False}

        def create():
            if not lib.fsdp_nvls_supported(dev.index):
                raise RuntimeError("no multicast/VMM support: " + _lib.last_error())
            if not _fd_passing_ok():
                raise RuntimeError("no SCM_RIGHTS fd passing")
            check(lib.fsdp_comm_create_vmm(rank, world, pool_bytes, max_ctas,
                                           _lib.HANDLE_POSIX_FD, C.byref(h)), "comm_create_vmm")
            state["created"] = True

        def open_box():
            tokens: list = [None] * world
            dist.all_gather_object(tokens, os.urandom(8).hex(), group=group)
            state["box"] = _FdBox(tokens[0], rank)

        buf = (C.c_char * _lib.SHAREABLE_BYTES)()

        def export_pool():
            check(lib.fsdp_comm_export_pool(h, buf), "comm_export_pool")
            state["own_fd"] = int.from_bytes(bytes(buf)[:4], "little", signed=True)

        def import_pools():
            got = state["box"].exchange({p: state["own_fd"] for p in range(world) if p != rank},
                                        world - 1, tag=0)
            try:
                for p, fd in got.items():
                    check(lib.fsdp_comm_import_pool(h, p, _handle_bytes(fd)), "comm_import_pool")
            finally:
                for fd in got.values():
                    os.close(fd)

        leader = rank // F * F

        def create_mc():
            if rank == leader:
                check(lib.fsdp_nvls_create(h, F, buf), "nvls_create")
                state["mc_fd"] = int.from_bytes(bytes(buf)[:4], "little", signed=True)

        def import_mc():
            sends = ({p: state["mc_fd"] for p in range(leader + 1, leader + F)}
                     if rank == leader else {})
            got = state["box"].exchange(sends, 0 if rank == leader else 1, tag=1)
            try:
                if rank != leader:
                    check(lib.fsdp_nvls_import(h, F, _handle_bytes(got[leader])), "nvls_import")
            finally:
                for fd in got.values():
                    os.close(fd)

        phases = [create, open_box, export_pool, import_pools, create_mc, import_mc,
                  lambda: check(lib.fsdp_nvls_add_device(h), "nvls_add_device"),
                  lambda: check(lib.fsdp_nvls_bind(h), "nvls_bind")]
        ok, err = True, ""
        for i, ph in enumerate(phases):
            ok, err = attempt(ph)
            if not ok:
                break
            if ph is open_box:
                dist.barrier(group=group)              # every box is listening
        if state["box"] is not None:
            state["box"].close()
        for k in ("own_fd", "mc_fd"):
            if state[k] >= 0:
                os.close(state[k])
        torch.cuda.synchronize()
        dist.barrier(group=group)
        if not ok:
            if state["created"]:
                lib.fsdp_comm_destroy(h)
            cls.last_nvls_error = err
            return None
        return cls(h.value, rank, world, False, dev)

    last_nvls_error = ""

    @property
    def nvls_group(self) -> int:
        """Size of the shard group bound to an NVLS multicast object (0: none)."""
        return int(lib.fsdp_nvls_group_size(self._h))

    @classmethod
    def create_emulated(cls, world: int, pool_bytes: int, max_ctas: int = 16) -> "DeviceComm":
        dev = torch.device("cuda", torch.cuda.current_device())
        h = C.c_void_p()
        check(lib.fsdp_comm_create_emulated(world, pool_bytes, max_ctas, C.byref(h)),
              "comm_create_emulated")
        return cls(h.value, 0, world, True, dev)

    def close(self) -> None:
        if not self.closed:
            torch.cuda.synchronize(self.device)
            self._pools = []
            lib.fsdp_comm_destroy(self._h)
            self.closed = True

    def set_timeout_ms(self, ms: int) -> None:
        check(lib.fsdp_comm_set_timeout_ms(self._h, int(ms)))

    KIND_AG, KIND_RS, KIND_AR = 0, 1, 2

    def set_mode(self, split: bool = True, timing: bool = False) -> None:
        """split: 1-CTA enter/exit barrier kernels around signal-only data
        kernels (default); timing: CUDA events around every data kernel."""
        check(lib.fsdp_comm_set_mode(self._h, int(split), int(timing)))

    def set_ctas(self, kind: int, ctas: int) -> None:
        """Grid cap of one collective kind's data kernel (same on every rank)."""
        check(lib.fsdp_comm_set_ctas(self._h, kind, int(ctas)))

    def timing_drain(self, kind: int) -> list[float]:
        """Durations (ms) of the data kernels of `kind` since the last drain."""
        buf = (C.c_float * 65536)()
        cnt = C.c_int(0)
        check(lib.fsdp_comm_timing_drain(self._h, kind, buf, 65536, C.byref(cnt)))
        return [buf[i] for i in range(min(cnt.value, 65536))]

    # -------------------------------------------------------------- memory --
    @property
    def nranks_local(self) -> int:
        return self.world if self.emulated else 1

    def alloc(self, nbytes: int, align: int = 256) -> int:
        """Symmetric region: same offset on every rank for the same call order."""
        off = (self._cursor + align - 1) // align * align
        if off + nbytes > self.pool_bytes:
            raise MemoryError(f"symmetric pool exhausted: need {off + nbytes} of {self.pool_bytes} B")
        self._cursor = off + nbytes
        return off

    def view(self, offset: int, numel: int, dtype: torch.dtype, e: int = 0) -> torch.Tensor:
        """Tensor over [offset, offset + numel*itemsize) of local pool `e`."""
        nb = numel * _ES[dtype]
        return self._pools[e][offset: offset + nb].view(dtype)

    def device_error(self) -> int:
        return int(lib.fsdp_comm_device_error(self._h))

    def fold_error(self, flag: torch.Tensor | None, keep: bool, mirror: torch.Tensor | None = None,
                   stream=None) -> None:
        """On `stream`: flag = 1 if the error word is set, else (keep ? flag : 0);
        the word is also mirrored into `mirror` (pinned int32 host tensor)."""
        check(lib.fsdp_comm_fold_error(self._h, flag.data_ptr() if flag is not None else None,
                                       int(keep), mirror.data_ptr() if mirror is not None else None,
                                       stream_ptr(stream)), "comm_fold_error")

    def set_fault(self, misorder_reduce_scatter: bool) -> None:
        """Verify-sensitivity fault hook (collectives.py:296): member k of every
        reduce-scatter receives chunk (k + 1) % size."""
        check(lib.fsdp_comm_set_fault(self._h, int(misorder_reduce_scatter)), "comm_set_fault")

    def clear_error(self) -> None:
        check(lib.fsdp_comm_clear_error(self._h), "comm_clear_error")

    _CH_NAMES = {0: "AG", 1: "RS", 2: "AR", 3: "SCALAR"}

    def timeout_info(self) -> dict | None:
        """Where this rank's first local timeout happened (None if none here:
        the abort came from a peer)."""
        buf = (C.c_uint32 * 6)()
        check(lib.fsdp_comm_timeout_info(self._h, buf), "comm_timeout_info")
        v = list(buf)
        if not v[0]:
            return None
        info = {"epoch": v[3], "channel": self._CH_NAMES.get(v[4], v[4]), "group": (v[5] >> 8, v[5] & 255),
                "seen": v[2]}
        flag_words = 4 * 3 * _lib.MAX_RANKS * _lib.MAX_CTAS
        w = v[1]
        if w < flag_words:
            cta = w % _lib.MAX_CTAS
            src = (w // _lib.MAX_CTAS) % _lib.MAX_RANKS
            ph = (w // (_lib.MAX_CTAS * _lib.MAX_RANKS)) % 3
            info.update(waiting_for_rank=src, phase=("enter", "data/exit", "phase2")[ph] if cta != _lib.MAX_CTAS - 1
                        else "enter", slot=cta)
        else:
            info.update(ll_line_byte_offset=w * 4)
        return info

    def raise_device_error(self) -> None:
        err = self.device_error()
        if err == _lib.E_TIMEOUT:
            info = self.timeout_info()
            where = (f" (here: channel {info['channel']} epoch {info['epoch']} group {info['group']}, "
                     f"{ {k: v for k, v in info.items() if k not in ('channel', 'epoch', 'group')} })"
                     if info else " (aborted by a peer)")
            raise DeadlockError("a cross-GPU collective wait timed out on device: some group member "
                                "never entered the matching collective" + where)
        if err:
            raise RuntimeError(f"device error word = {err}")

    # --------------------------------------------------------- collectives --
    def _ptrs(self, ts: Sequence[torch.Tensor]):
        if len(ts) != self.nranks_local:
            raise CollectiveError(f"expected {self.nranks_local} per-rank buffers, got {len(ts)}")
        return _lib.ptr_array([t.data_ptr() for t in ts])

    def all_gather(self, gdesc, shards: Sequence[torch.Tensor], dst_off: int, dst_dtype: torch.dtype,
                   stream=None, channel: int = _lib.CH_AG) -> None:
        n = shards[0].numel()
        check(lib.fsdp_allgather(self._h, channel, gdesc[0], gdesc[1], self._ptrs(shards),
                                 dtype_code(shards[0].dtype), n, dst_off, dtype_code(dst_dtype),
                                 stream_ptr(stream)), "allgather")

    def reduce_scatter(self, gdesc, flats: Sequence[torch.Tensor], stage_off: int,
                       outs: Sequence[torch.Tensor], prediv: float = 1.0, postdiv: float = 1.0,
                       accumulate: bool = False, stream=None, channel: int = _lib.CH_RS) -> None:
        n = outs[0].numel()
        check(lib.fsdp_reduce_scatter(self._h, channel, gdesc[0], gdesc[1], self._ptrs(flats),
                                      dtype_code(flats[0].dtype), n, stage_off, self._ptrs(outs),
                                      float(prediv), float(postdiv), int(accumulate),
                                      stream_ptr(stream)), "reduce_scatter")

    def reduce_scatter_pull(self, gdesc, src_off: int, src_dtype: torch.dtype,
                            outs: Sequence[torch.Tensor], prediv: float = 1.0, postdiv: float = 1.0,
                            accumulate: bool = False, stream=None, channel: int = _lib.CH_RS,
                            tma: bool = True) -> None:
        """Payload already in every member's pool at `src_off` (gsize*n elems)."""
        n = outs[0].numel()
        fn = lib.fsdp_reduce_scatter_tma if tma else lib.fsdp_reduce_scatter_pull
        check(fn(self._h, channel, gdesc[0], gdesc[1], src_off,
                                           dtype_code(src_dtype), n, self._ptrs(outs), float(prediv),
                                           float(postdiv), int(accumulate), stream_ptr(stream)),
              "reduce_scatter_pull")

    def all_gather_ce(self, gdesc, shard: torch.Tensor, dst_off: int, stream=None,
                      channel: int = _lib.CH_AG) -> None:
        """Copy-engine all-gather (same dtype in and out)."""
        check(lib.fsdp_allgather_ce(self._h, channel, gdesc[0], gdesc[1], shard.data_ptr(),
                                    dtype_code(shard.dtype), shard.numel(), dst_off,
                                    stream_ptr(stream)), "allgather_ce")

    def all_gather_nvls(self, gdesc, shard: torch.Tensor, dst_off: int, dst_dtype: torch.dtype,
                        stream=None, channel: int = _lib.CH_AG) -> None:
        """NVLS multicast all-gather (fused cast); same contract as all_gather,
        falls back to it inside the library when the group is not the bound one."""
        check(lib.fsdp_allgather_nvls(self._h, channel, gdesc[0], gdesc[1], shard.data_ptr(),
                                      dtype_code(shard.dtype), shard.numel(), dst_off,
                                      dtype_code(dst_dtype), stream_ptr(stream)), "allgather_nvls")

    def reduce_scatter_ce(self, gdesc, src_off: int, src_dtype: torch.dtype, stage_off: int,
                          out: torch.Tensor, prediv: float = 1.0, postdiv: float = 1.0,
                          accumulate: bool = False, stream=None, channel: int = _lib.CH_RS) -> None:
        """Copy-engine pull of the peers' chunks + local ascending fp32 reduction
        (`out` fp32, or bf16: the sum rounded once, no accumulate)."""
        check(lib.fsdp_reduce_scatter_ce_out(self._h, channel, gdesc[0], gdesc[1], src_off,
                                             dtype_code(src_dtype), out.numel(), stage_off,
                                             out.data_ptr(), dtype_code(out.dtype), float(prediv),
                                             float(postdiv), int(accumulate), stream_ptr(stream)),
              "reduce_scatter_ce")

    def all_reduce(self, gdesc, ins: Sequence[torch.Tensor], stage_off: int, gather_off: int,
                   outs: Sequence[torch.Tensor], postdiv: float = 1.0, accumulate: bool = False,
                   stream=None, channel: int = _lib.CH_AR) -> None:
        n = ins[0].numel()
        check(lib.fsdp_allreduce(self._h, channel, gdesc[0], gdesc[1], self._ptrs(ins),
                                 dtype_code(ins[0].dtype), n, stage_off, gather_off,
                                 self._ptrs(outs), float(postdiv), int(accumulate),
                                 stream_ptr(stream)), "allreduce")

    @staticmethod
    def ll_bytes(gsize: int, n: int, dtype: torch.dtype) -> int:
        """Size of the LL region a (gsize, n, dtype) low-latency collective uses."""
        return int(lib.fsdp_ll_bytes(gsize, n, dtype_code(dtype)))

    def all_gather_ll(self, gdesc, shards: Sequence[torch.Tensor], dst_off: int,
                      dst_dtype: torch.dtype, ll_off: int, stream=None,
                      channel: int = _lib.CH_AG) -> None:
        """One-kernel low-latency all-gather (same result as all_gather)."""
        n = shards[0].numel()
        check(lib.fsdp_allgather_ll(self._h, channel, gdesc[0], gdesc[1], self._ptrs(shards),
                                    dtype_code(shards[0].dtype), n, dst_off, dtype_code(dst_dtype),
                                    ll_off, stream_ptr(stream)), "allgather_ll")

    def reduce_scatter_ll(self, gdesc, flats: Sequence[torch.Tensor], ll_off: int,
                          outs: Sequence[torch.Tensor], prediv: float = 1.0, postdiv: float = 1.0,
                          accumulate: bool = False, stream=None, channel: int = _lib.CH_RS) -> None:
        """One-kernel low-latency reduce-scatter (same result as reduce_scatter)."""
        n = outs[0].numel()
        check(lib.fsdp_reduce_scatter_ll(self._h, channel, gdesc[0], gdesc[1], self._ptrs(flats),
                                         dtype_code(flats[0].dtype), n, ll_off, self._ptrs(outs),
                                         float(prediv), float(postdiv), int(accumulate),
                                         stream_ptr(stream)), "reduce_scatter_ll")

    def all_reduce_ce(self, gdesc, inp: torch.Tensor, stage_off: int, gather_off: int,
                      out: torch.Tensor, postdiv: float = 1.0, accumulate: bool = False,
                      stream=None, channel: int = _lib.CH_AR) -> None:
        """Copy-engine all-reduce (same bits as all_reduce; real communicator)."""
        check(lib.fsdp_allreduce_ce(self._h, channel, gdesc[0], gdesc[1], inp.data_ptr(),
                                    dtype_code(inp.dtype), inp.numel(), stage_off, gather_off,
                                    out.data_ptr(), float(postdiv), int(accumulate),
                                    stream_ptr(stream)), "allreduce_ce")

    def all_reduce_ce_pool(self, gdesc, inp: torch.Tensor, stage_off: int, out_off: int,
                           postdiv: float = 1.0, stream=None, channel: int = _lib.CH_AR) -> None:
        """Copy-engine all-reduce whose output is the pool region at out_off
        (same offset on every member): no gather buffer, no epilogue."""
        check(lib.fsdp_allreduce_ce_pool(self._h, channel, gdesc[0], gdesc[1], inp.data_ptr(),
                                         dtype_code(inp.dtype), inp.numel(), stage_off, out_off,
                                         float(postdiv), stream_ptr(stream)), "allreduce_ce_pool")

    def scalar_all_reduce(self, ins: Sequence[torch.Tensor], outs: Sequence[torch.Tensor],
                          stream=None) -> None:
        check(lib.fsdp_allreduce_scalar(self._h, self._ptrs(ins), self._ptrs(outs),
                                        stream_ptr(stream)), "allreduce_scalar")

    @staticmethod
    def ar_staging_elems(n: int, gsize: int) -> int:
        c = -(-n // gsize)
        c = -(-c // 8) * 8
        return c * gsize


class DeviceFabric:
    """shardsim-shaped collectives on device tensors (collectives.py:183-306).

    Each call validates the reference's entry contract synchronously and
    returns the result tensor(s).  For an emulated communicator the `local`
    argument is a list with one tensor per rank and so is the result."""

    def __init__(self, comm: DeviceComm, scratch_bytes: int):
        self.comm = comm
        self.scratch_bytes = scratch_bytes
        self.off_a = comm.alloc(scratch_bytes)
        self.off_b = comm.alloc(scratch_bytes)

    def _norm(self, rank: int, group: Sequence[int], local, kind: str):
        group = tuple(sorted(group))
        if rank not in group:
            raise CollectiveError(f"rank {rank} is not a member of {group}")
        locs = list(local) if isinstance(local, (list, tuple)) else [local]
        for t in locs:
            if t.dim() != 1:
                raise CollectiveError(f"{kind}: expected a flat 1-d buffer, got shape {tuple(t.shape)}")
        if len({t.numel() for t in locs}) > 1:
            raise CollectiveError(f"{kind} on group {group}: uneven inputs are rejected, pad explicitly")
        return group, locs

    def all_gather(self, rank, group, local, stream=None):
        group, locs = self._norm(rank, group, local, "AG")
        gd = group_desc_of(group, self.comm.world)
        n = locs[0].numel()
        nb = n * gd[0] * _ES[locs[0].dtype]
        if nb > self.scratch_bytes:
            raise CollectiveError("AG larger than the fabric scratch region")
        self.comm.all_gather(gd, locs, self.off_a, locs[0].dtype, stream)
        outs = [self.comm.view(self.off_a, n * gd[0], locs[0].dtype, e).clone()
                for e in range(self.comm.nranks_local)]
        return outs if isinstance(local, (list, tuple)) else outs[0]

    def reduce_scatter(self, rank, group, local, stream=None):
        group, locs = self._norm(rank, group, local, "RS")
        gd = group_desc_of(group, self.comm.world)
        length = locs[0].numel()
        if length % gd[0]:
            raise CollectiveError(f"reduce_scatter: input length {length} not divisible by group size {gd[0]}")
        n = length // gd[0]
        outs = [torch.empty(n, dtype=torch.float32, device=self.comm.device) for _ in locs]
        self.comm.reduce_scatter(gd, locs, self.off_a, outs, stream=stream)
        return outs if isinstance(local, (list, tuple)) else outs[0]

    def all_reduce(self, rank, group, local, stream=None):
        group, locs = self._norm(rank, group, local, "AR")
        gd = group_desc_of(group, self.comm.world)
        n = locs[0].numel()
        outs = [torch.empty(n, dtype=torch.float32, device=self.comm.device) for _ in locs]
        self.comm.all_reduce(gd, locs, self.off_a, self.off_b, outs, stream=stream)
        return outs if isinstance(local, (list, tuple)) else outs[0]
