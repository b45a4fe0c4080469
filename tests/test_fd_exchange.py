"""Host side of the NVLS / VMM setup on CPU: the file-descriptor exchange
between rank processes (SCM_RIGHTS over abstract Unix sockets) that carries
the cuMemExportToShareableHandle POSIX fds.  Three real processes (gloo for
the token broadcast): every rank sends a descriptor of its own temp file to
every peer (the pool round), then rank 0 sends one more to the others (the
multicast-object round); each receiver reads the peer's file through the
received descriptor."""
import os
import socket
import sys
import tempfile

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tmp, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2304_11277_b200.comm import _FdBox, _handle_bytes
        tokens = [None] * world
        dist.all_gather_object(tokens, os.urandom(8).hex())
        box = _FdBox(tokens[0], rank)
        path = os.path.join(tmp, f"pool{rank}")
        with open(path, "w") as fh:
            fh.write(f"pool of rank {rank}")
        own = os.open(path, os.O_RDONLY)
        dist.barrier()
        got = box.exchange({p: own for p in range(world) if p != rank}, world - 1, tag=0)
        seen = {}
        for p, fd in got.items():
            seen[p] = os.pread(fd, 64, 0).decode()
            assert int.from_bytes(_handle_bytes(fd)[:4], "little", signed=True) == fd
            os.close(fd)
        assert seen == {p: f"pool of rank {p}" for p in range(world) if p != rank}, seen
        mc = -1
        if rank == 0:
            mpath = os.path.join(tmp, "mc")
            with open(mpath, "w") as fh:
                fh.write("multicast object")
            mc = os.open(mpath, os.O_RDONLY)
        dist.barrier()
        got = box.exchange({p: mc for p in range(1, world)} if rank == 0 else {},
                           0 if rank == 0 else 1, tag=1)
        if rank != 0:
            assert list(got) == [0]
            assert os.pread(got[0], 64, 0).decode() == "multicast object"
            os.close(got[0])
        box.close()
        os.close(own)
        if mc >= 0:
            os.close(mc)
        dist.barrier()
        q.put((rank, "ok"))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_fd_exchange_three_ranks():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    with tempfile.TemporaryDirectory() as tmp:
        procs = [ctx.Process(target=_worker, args=(r, world, port, tmp, q))
                 for r in range(world)]
        for p in procs:
            p.start()
        res = dict(q.get(timeout=120) for _ in range(world))
        for p in procs:
            p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res

