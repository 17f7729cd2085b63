"""In-process block transport for the reference-compatible exchange API.

The reference's partitioned mode moves numpy blocks between part threads
through per-pair FIFO queues (transport.py:42-95). On the device path the
redistribution is a device-side copy (one GPU) or an NCCL all-to-all
(``distributed``), so this module only keeps the host-side contract for
callers of ``exchange_forward`` / ``exchange_inverse``. The TCP frame codec
(transport.py:98-240) is multi-host plumbing and out of scope.
"""

import queue

from .errors import ExchangeError

STAGE_FORWARD = 1
STAGE_INVERSE = 2


class InProcessTransport:
    """One part's endpoint of an InProcessMesh."""

    def __init__(self, mesh, part):
        self._mesh = mesh
        self.part = part

    def send(self, to_part, stage, block):
        if to_part == self.part:
            raise ExchangeError("self-send is a local copy, not a transfer",
                                sender=self.part, receiver=to_part)
        self._mesh.channel(self.part, to_part).put((stage, block))

    def receive(self, from_part, stage, extents):
        edge = (from_part, self.part)
        try:
            got, block = self._mesh.channel(*edge).get(timeout=self._mesh.timeout)
        except queue.Empty:
            raise ExchangeError(f"timed out waiting for block {from_part} -> {self.part}",
                                sender=from_part, receiver=self.part) from None
        if got != stage:
            raise ExchangeError(f"stage mismatch on edge {edge}: expected {stage}, got {got}",
                                sender=from_part, receiver=self.part)
        n_z, n_y, n_x = block.shape
        if (n_x, n_y, n_z) != tuple(extents):
            raise ExchangeError(f"block extents {(n_x, n_y, n_z)} != expected {tuple(extents)} "
                                f"on edge {edge}", sender=from_part, receiver=self.part)
        return block

    def close(self):
        pass


class InProcessMesh:
    """All-pairs FIFO channels between n_parts endpoints."""

    def __init__(self, n_parts, timeout=60.0):
        self.n_parts = n_parts
        self.timeout = timeout
        self._channels = {(s, r): queue.Queue() for s in range(n_parts)
                          for r in range(n_parts) if s != r}

    def channel(self, sender, receiver):
        return self._channels[(sender, receiver)]

    def endpoint(self, part) -> InProcessTransport:
        return InProcessTransport(self, part)
