"""Row-partitioned power iteration.

One process per GPU. The matrix is row-partitioned, balanced by nnz
(spmv_dist_partition, C ABI); each rank owns a row slab whose global column
indices are remapped into a padded all-gather layout (spmv_dist_remap_columns)
so x is replicated by a single all_gather_into_tensor per step with no
compaction pass. Per step k:

    z_k(local) = alpha_k · A_local · z_{k-1},  alpha_k = 1/sqrt(S_{k-1})   [spmv_power_step, one kernel]
    (S_k, D_k) = all_reduce(Σ z_k², Σ z_{k-1}(own rows)·z_k)              [8·2 bytes]
    z_k(full)  = all_gather(z_k(local))                                    [NCCL over NVLink]
    lambda_k   = D_k / sqrt(S_{k-1})

The SpMV and its fused norm epilogue run in libspmv.so kernels; torch.distributed
(NCCL on GPUs, gloo in the CPU tests) only moves the vector and the two sums.
`local_step` / `local_norm2` are injectable so the CPU tests can drive this
exact loop with another local implementation.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Layout:
    """Padded all-gather layout of a row partition."""
    bounds: np.ndarray  # int64 [world+1], global row bounds
    world: int
    chunk: int          # max rows per rank

    @classmethod
    def from_bounds(cls, bounds):
        b = np.asarray(bounds, np.int64)
        world = b.shape[0] - 1
        chunk = int(np.max(np.diff(b))) if world > 0 else 0
        return cls(b, world, max(chunk, 1))

    def rows_of(self, rank):
        return int(self.bounds[rank]), int(self.bounds[rank + 1])

    @property
    def padded_n(self):
        return self.world * self.chunk

    def to_padded(self, v_global, xp=np):
        """Global vector -> padded layout (host numpy or torch)."""
        out = xp.zeros(self.padded_n, dtype=v_global.dtype) if xp is np else None
        if xp is np:
            for r in range(self.world):
                a, b = self.rows_of(r)
                out[r * self.chunk: r * self.chunk + (b - a)] = v_global[a:b]
            return out
        raise TypeError

    def from_padded(self, v_padded):
        parts = [v_padded[r * self.chunk: r * self.chunk + (self.rows_of(r)[1] - self.rows_of(r)[0])]
                 for r in range(self.world)]
        if isinstance(v_padded, np.ndarray):
            return np.concatenate(parts)
        import torch
        return torch.cat(parts)


class PowerIteration:
    """Drives E power steps over a row slab with torch.distributed collectives.

    local_step(x_full, y_local, sums_prev, sums_out, row_offset) computes the
    slab's z_k and its two partial sums; local_norm2(x_local, sums_out)
    computes Σ x_local². Both are the C-ABI calls on the GPU path."""

    def __init__(self, layout: Layout, rank: int, local_step, local_norm2, group=None, halo=None):
        import torch.distributed as dist
        self.layout = layout
        self.rank = rank
        self.local_step = local_step
        self.local_norm2 = local_norm2
        self.group = group
        self.halo = halo  # HaloExchange: exchange only the referenced remote entries
        self.dist = dist if (dist.is_available() and dist.is_initialized() and layout.world > 1) else None

    def _allreduce(self, t):
        if self.dist is not None:
            self.dist.all_reduce(t, group=self.group)

    def _allgather(self, full, local_chunk):
        if self.dist is not None:
            self.dist.all_gather_into_tensor(full, local_chunk, group=self.group)
        else:
            full.copy_(local_chunk)

    def run(self, x_full, steps: int, bufs=None, on_step=None):
        """x_full: padded global start vector z_0 (any nonzero norm), torch
        tensor on this rank's device. Returns (z_final_full, lambdas(list of
        device scalars), sums list). Buffers may be passed to avoid allocation."""
        import torch
        L = self.layout
        dev = x_full.device
        a, b = L.rows_of(self.rank)
        nloc = b - a
        if bufs is None:
            bufs = self.make_buffers(x_full.dtype, dev, steps)
        cur, nxt, chunk_buf, sums = bufs["cur"], bufs["nxt"], bufs["chunk"], bufs["sums"]
        cur.copy_(x_full)
        # S_0 = ||z_0||² (global)
        self.local_norm2(cur[self.rank * L.chunk: self.rank * L.chunk + nloc], sums[0])
        self._allreduce(sums[0])
        for k in range(steps):
            if self.dist is None and L.world == 1:
                # single rank: the SpMV writes the next iterate in place (no gather)
                self.local_step(cur, nxt[:nloc], sums[k], sums[k + 1], 0)
            else:
                y_local = chunk_buf[:nloc]
                self.local_step(cur, y_local, sums[k], sums[k + 1], self.rank * L.chunk)
                self._allreduce(sums[k + 1])
                if self.halo is not None:
                    nxt[self.rank * L.chunk: self.rank * L.chunk + nloc] = y_local
                    self.halo.exchange(nxt)
                else:
                    self._allgather(nxt, chunk_buf)
            cur, nxt = nxt, cur
            if on_step is not None:
                on_step(k)
        bufs["cur"], bufs["nxt"] = cur, nxt
        return cur, sums

    def make_buffers(self, dtype, device, steps):
        import torch
        L = self.layout
        return {"cur": torch.zeros(L.padded_n, dtype=dtype, device=device),
                "nxt": torch.zeros(L.padded_n, dtype=dtype, device=device),
                "chunk": torch.zeros(L.chunk, dtype=dtype, device=device),
                "sums": torch.zeros(steps + 1, 2, dtype=torch.float64, device=device)}

    @staticmethod
    def lambdas(sums):
        """lambda_k = D_k / sqrt(S_{k-1}) for k = 1..steps (host numpy)."""
        s = sums.detach().cpu().numpy() if hasattr(sums, "detach") else np.asarray(sums)
        return s[1:, 1] / np.sqrt(s[:-1, 0])


class HaloExchange:
    """Point-to-point exchange of exactly the remote entries of x a row slab
    references — the torch.distributed mirror of the native plan's
    SPMV_PLAN_HALO lists (plan.cu build_halo_lists / exchange_step):
    sorted unique remote padded positions grouped by owner; counts all-gathered
    once; request lists sent to the owners once; per step each owner sends the
    requested values and the receiver scatters them into its vector."""

    def __init__(self, layout: Layout, rank: int, slab_cols, group=None):
        import torch
        import torch.distributed as dist
        L = layout
        a, b = L.rows_of(rank)
        lo, hi = rank * L.chunk, rank * L.chunk + (b - a)
        cols = np.asarray(slab_cols, np.int64)
        remote = np.unique(cols[(cols < lo) | (cols >= hi)])
        owner = remote // L.chunk
        self.need = {int(q): remote[owner == q] for q in np.unique(owner)}
        counts = torch.zeros(L.world, dtype=torch.int64)
        for q, v in self.need.items():
            counts[q] = len(v)
        allc = [torch.zeros(L.world, dtype=torch.int64) for _ in range(L.world)]
        dist.all_gather(allc, counts, group=group)
        give_cnt = {r: int(allc[r][rank]) for r in range(L.world) if int(allc[r][rank]) > 0}
        reqs, bufs = [], {}
        for q, v in self.need.items():
            reqs.append(dist.isend(torch.from_numpy(v.copy()), q, group=group))
        for r, c in give_cnt.items():
            bufs[r] = torch.empty(c, dtype=torch.int64)
            reqs.append(dist.irecv(bufs[r], r, group=group))
        for q in reqs:
            q.wait()
        self.give = {r: t for r, t in bufs.items()}
        self.need_t = {q: torch.from_numpy(v.copy()) for q, v in self.need.items()}
        self.group = group
        self.recv_elems = int(sum(len(v) for v in self.need.values()))

    def exchange(self, x_full):
        import torch
        import torch.distributed as dist
        reqs, bufs = [], {}
        for r, idx in self.give.items():
            reqs.append(dist.isend(x_full[idx].contiguous(), r, group=self.group))
        for q, idx in self.need_t.items():
            bufs[q] = torch.empty(len(idx), dtype=x_full.dtype)
            reqs.append(dist.irecv(bufs[q], q, group=self.group))
        for q in reqs:
            q.wait()
        for q, idx in self.need_t.items():
            x_full[idx] = bufs[q]


class NativeComm:
    """NCCL communicator of libspmv.so, bootstrapped through torch.distributed
    (rank 0 creates the unique id, a broadcast shares it)."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch
        import torch.distributed as dist
        from . import spmv_dist_init, spmv_dist_unique_id
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid = torch.frombuffer(bytearray(spmv_dist_unique_id()), dtype=torch.uint8).clone()
        if dist.is_initialized() and world > 1:
            t = uid.to(f"cuda:{device}") if dist.get_backend(group) == "nccl" else uid
            dist.broadcast(t, 0, group=group)
            uid = t.cpu()
        self.comm = spmv_dist_init(bytes(uid.numpy().tobytes()), rank, world, device)
        self.rank, self.world = rank, world

    def close(self):
        from . import spmv_dist_destroy
        if self.comm is not None:
            spmv_dist_destroy(self.comm)
            self.comm = None


def native_power_iteration(h, layout: Layout, rank: int, x0, bufs, steps: int, comm=None, time_kernels=False,
                           time_loop=False):
    """E power steps in one C-ABI call (loop + NCCL exchange in C++).
    Returns (z_E tensor view, sums, kernel_ms or None[, loop_ms])."""
    from . import spmv_power_iterate
    c = comm.comm if comm is not None else None
    fb, kms, lms = spmv_power_iterate(h, x0, bufs["cur"], bufs["nxt"], steps, bufs["sums"], c, layout.chunk,
                                      bufs["chunk"] if c is not None else None, time_kernels, time_loop)
    z = bufs["cur"] if fb == 0 else bufs["nxt"]
    if time_loop:
        return z, bufs["sums"], kms, lms
    return z, bufs["sums"], kms


def partition_rows(row_lengths, world):
    """nnz-balanced bounds via the C ABI (pure host integer logic)."""
    from . import spmv_dist_partition_lengths
    return spmv_dist_partition_lengths(np.asarray(row_lengths, np.int64), world)
