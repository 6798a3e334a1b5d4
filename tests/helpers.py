"""Shared helpers for parity tests."""

import numpy as np


def random_boxes(d, n, seed):
    """Same generator as oracle/make_golden.py:random_boxes."""
    rng = np.random.default_rng(seed)
    lengths = rng.uniform(0.01, 0.5, size=(n, d))
    lefts = rng.uniform(0.0, 1.0, size=(n, d)) * (1.0 - lengths)
    return lefts, lengths


def same_numpy_build(golden):
    return golden["numpy"] == np.__version__


def ulp_diff(a, b):
    """Distance in units-in-the-last-place between float64 arrays (same sign assumed)."""
    a = np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
    b = np.ascontiguousarray(b, dtype=np.float64).view(np.int64)
    return np.abs(a - b)


class ThreadComm:
    """In-process stand-in for sharded.Comm: `world` threads exchange through shared slots.
    Lets one GPU (or the CPU) run the SPMD drivers with several ranks."""

    class _Shared:
        def __init__(self, world):
            import threading
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world
            self.mail = {}

    def __init__(self, shared, rank):
        self._s, self.rank, self.world = shared, rank, shared.world

    @classmethod
    def make(cls, world):
        shared = cls._Shared(world)
        return [cls(shared, r) for r in range(world)]

    def allgather(self, a):
        self._s.slots[self.rank] = np.array(a, dtype=np.float64)
        self._s.barrier.wait()
        out = [x.copy() for x in self._s.slots]
        self._s.barrier.wait()
        return out

    def allreduce_sum(self, a):
        parts = self.allgather(a)
        total = parts[0].copy()
        for p in parts[1:]:
            total = total + p
        return total

    def barrier(self):
        self._s.barrier.wait()

    # ---- tensor-level collectives on CUDA tensors of ONE device (every rank a thread with its own library context and
    #      stream): the in-process stand-in for sharded.Comm's NCCL methods
    @staticmethod
    def _sync():
        import torch
        torch.cuda.current_stream().synchronize()

    def all_gather_into(self, out, inp):
        self._sync()                                   # my row is complete
        self._s.slots[self.rank] = inp
        self._s.barrier.wait()
        n = inp.numel()
        parts = [t.clone() for t in self._s.slots]     # read everyone (mine may alias `out`)
        self._sync()
        self._s.barrier.wait()                         # everyone has read: buffers may change again
        for r, t in enumerate(parts):
            out[r * n:(r + 1) * n].copy_(t)

    def _all_reduce(self, t, op):
        self._sync()
        self._s.slots[self.rank] = t
        self._s.barrier.wait()
        total = self._s.slots[0].clone()
        for other in self._s.slots[1:]:                # rank order on every rank: identical bits everywhere
            total = op(total, other)
        self._sync()
        self._s.barrier.wait()
        t.copy_(total)

    def all_reduce_sum_(self, t):
        import torch
        self._all_reduce(t, torch.add)

    def all_reduce_max_(self, t):
        import torch
        self._all_reduce(t, torch.maximum)

    def exchange_tensors(self, sends, recvs):
        self._sync()
        for r, t in sends.items():
            self._s.mail[(self.rank, r)] = t
        self._s.barrier.wait()
        for r, buf in recvs.items():
            buf.copy_(self._s.mail[(r, self.rank)])
        self._sync()
        self._s.barrier.wait()
        for r in sends:
            self._s.mail.pop((self.rank, r), None)
        self._s.barrier.wait()

    def exchange_rows(self, sends, recvs, d):
        for r, (lefts, lengths) in sends.items():
            self._s.mail[(self.rank, r)] = (np.array(lefts), np.array(lengths))
        self._s.barrier.wait()
        got = {r: self._s.mail[(r, self.rank)] for r in recvs}
        self._s.barrier.wait()
        for r in sends:
            self._s.mail.pop((self.rank, r), None)
        self._s.barrier.wait()
        return got


def run_ranks(world, fn):
    """Run fn(rank, comm) on `world` threads; returns the list of results, re-raising the first failure."""
    import threading
    comms = ThreadComm.make(world)
    out, err = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r, comms[r])
        except BaseException as exc:  # noqa: BLE001
            err.append(exc)
            comms[r]._s.barrier.abort()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if err:
        raise err[0]
    return out
