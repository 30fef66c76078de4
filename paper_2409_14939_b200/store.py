"""Host-resident feature tables for the Match loader (config 4 of
BASELINE.json: papers100M-shaped features in pinned host memory).

The loader (loader.cu ``fgl_gather_rows_cached``) reads the delta rows of
every batch zero-copy over the host link, so the table must be page-locked
and mapped.  With data parallelism every rank of the node reads
the SAME table: rank 0 allocates it once in an anonymous shared-memory file
(``memfd``), every rank maps that file and page-locks its mapping
(``fgl_host_register``), so eight ranks need one 56.8 GB copy, not eight.
Rows are ``ld = round_up(d, 4)`` floats so each is 16-byte aligned.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib

__all__ = ["HostFeatureStore"]


class HostFeatureStore:
    """A pinned, device-mapped [num_nodes, ld] f32 feature table in host memory.

    ``table`` is the host tensor (valid CPU tensor), ``dev_ptr`` the address
    the kernels read it through, ``dim`` the logical feature width."""

    def __init__(self, table, dim: int, dev_ptr: int, registered: bool, fd: int | None = None):
        self.table = table
        self.dim = int(dim)
        self.ld = int(table.shape[1])
        self.num_nodes = int(table.shape[0])
        self.dev_ptr = int(dev_ptr)
        self._registered = registered
        self._fd = fd

    @property
    def shape(self):
        return (self.num_nodes, self.dim)

    @staticmethod
    def _ld(d):
        return (int(d) + 3) // 4 * 4

    @classmethod
    def private(cls, feats) -> "HostFeatureStore":
        """A process-private pinned copy of `feats` ([N, d] tensor or array)."""
        import torch
        ft = feats if isinstance(feats, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(feats, np.float32))
        n, d = int(ft.shape[0]), int(ft.shape[1])
        host = torch.zeros((n, cls._ld(d)), dtype=torch.float32).pin_memory()
        host[:, :d].copy_(ft.cpu() if ft.is_cuda else ft)
        # cudaHostAlloc memory is mapped; with UVA its host address is the device address
        return cls(host, d, host.data_ptr(), registered=False)

    @classmethod
    def shared(cls, num_nodes: int, dim: int, fill=None, *, rank: int = 0, world: int = 1) -> "HostFeatureStore":
        """One table for all ranks of the node.  Rank 0 creates an anonymous
        shared-memory file of N x ld floats and calls ``fill(table)`` (a CPU
        tensor view of [N, ld]); the path is broadcast over the process group
        and every rank maps and page-locks the same pages.  Collective over
        the default process group when world > 1."""
        import torch
        n, d = int(num_nodes), int(dim)
        ld = cls._ld(d)
        nbytes = n * ld * 4
        fd = None
        path = [None]
        if rank == 0:
            fd = os.memfd_create("fgl_features")
            os.ftruncate(fd, nbytes)
            path[0] = f"/proc/{os.getpid()}/fd/{fd}"
        if world > 1:
            import torch.distributed as dist
            dist.broadcast_object_list(path, src=0)
        flat = torch.from_file(path[0], shared=True, size=n * ld, dtype=torch.float32)
        table = flat.view(n, ld)
        if rank == 0 and fill is not None:
            fill(table)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        dev = ctypes.c_void_p()
        _lib.call("fgl_host_register", table.data_ptr(), nbytes, ctypes.byref(dev))
        return cls(table, d, dev.value, registered=True, fd=fd)

    def close(self):
        if self._registered:
            try:
                _lib.lib().fgl_host_unregister(self.table.data_ptr())
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass
            self._registered = False
        if self._fd is not None:
            try:
                os.close(self._fd)
            except OSError:
                pass
            self._fd = None

    def __del__(self):
        self.close()
