"""Single-process emulation of the sharded drivers' collectives (TEST
INFRASTRUCTURE): one thread per shard, all on one GPU; allgather /
allreduce exchange device tensors through shared slots between two
barriers.  Every thread launches on the legacy default stream, so a
consumer's kernels are ordered after the producers' (no kernel waits on
another)."""

import threading

import torch


class ThreadComm:
    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.barrier = threading.Barrier(world)

    def for_rank(self, rank):
        return _RankComm(self, rank)


class _RankComm:
    def __init__(self, hub, rank):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def _exchange(self, x):
        self.hub.slots[self.rank] = x.reshape(-1).clone()
        self.hub.barrier.wait()
        parts = list(self.hub.slots)
        self.hub.barrier.wait()
        return parts

    def allgather(self, x):
        return torch.cat(self._exchange(x))

    def allreduce_sum(self, x):
        parts = self._exchange(x)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc += p
        x.copy_(acc.reshape(x.shape))
        return x


def run_ranks(world, fn):
    """Run fn(rank, comm) on `world` threads; returns the results by rank."""
    hub = ThreadComm(world)
    out, err = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r, hub.for_rank(r))
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err.append(e)
            hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out
