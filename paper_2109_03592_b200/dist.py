"""Multi-GPU PCG: one process per GPU, elements partitioned by partition_rcb.

torch.distributed is plumbing only: it gathers the 136-byte peer-window blobs
once at setup (all_gather_object) and provides the benchmark barrier/max.
The per-iteration exchanges -- shared-node copy values and the CG scalars --
are stores from our own kernels into the peers' CUDA-IPC windows over NVLink
(paper_2109_03592_b200/csrc/dist_kern.cuh), not collectives.

    import torch.distributed as dist
    dist.init_process_group("nccl")
    ctx = DistContext.box(64, 64, 64, 7, deform=0.05, device=local_rank)
    op = HelmholtzOperator(ctx)
    res = pcg(op, b_local, x_local, KrylovConfig(1e-8, 5000))   # same API as 1 GPU
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .api import Context, _check, build_box_mesh, partition_rcb

lib = L.lib


def _box_desc(ex, ey, ez, degree, periodic, deform, origin, lengths):
    d = L.BoxDesc()
    d.ex, d.ey, d.ez, d.degree = ex, ey, ez, degree
    for q in range(3):
        d.periodic[q] = int(bool(periodic[q]))
        d.origin[q] = origin[q]
        d.lengths[q] = lengths[q]
    d.deform_amplitude = float(deform)
    return d


def plan(ex, ey, ez, degree, rank_of, nranks, rank, periodic=(False, False, False)):
    """Host-only exchange plan of one rank (no GPU); numpy arrays by name."""
    d = _box_desc(ex, ey, ez, degree, periodic, 0.0, (0, 0, 0), (1, 1, 1))
    h = C.c_void_p()
    rank_of = np.ascontiguousarray(rank_of, np.int32)
    _check(lib.sbx_dist_plan_create(C.byref(d), rank_of.ctypes.data, nranks, rank, C.byref(h)))
    try:
        sz = np.zeros(9, np.int64)
        _check(lib.sbx_dist_plan_sizes(h, sz.ctypes.data))
        EL, NL, nb, nbc, ni, nic, nq, rt, st = (int(v) for v in sz)

        def arr(which, count, dtype):
            a = np.zeros(max(count, 1), dtype)
            _check(lib.sbx_dist_plan_array(h, which, a.ctypes.data))
            return a[:count]

        out = {
            "loc_elems": arr(0, EL, np.int64), "nodes_local": NL,
            "b_off": arr(1, nb + 1, np.int32), "b_idx": arr(2, nbc, np.int32),
            "if_off": arr(3, ni + 1, np.int32), "if_code": arr(4, nic, np.int32),
            "nbr": arr(5, nq, np.int32), "send_count": arr(6, nq, np.int64),
            "send_idx": arr(7, st, np.int32), "recv_count": arr(8, nq, np.int64),
            "recv_base": arr(9, nq, np.int64), "nbr27": arr(10, EL * 27, np.int32),
            "inv_mult": arr(11, NL, np.float64), "mask": arr(12, NL, np.float64),
            "if_gid": arr(13, ni, np.int64), "recv_total": rt,
        }
    finally:
        lib.sbx_dist_plan_destroy(h)
    return out


class DistContext(Context):
    """This rank's part of a structured box on its GPU, connected to its peers."""

    @classmethod
    def box(cls, ex, ey, ez, degree, deform=0.0, periodic=(False, False, False),
            origin=(0.0, 0.0, 0.0), lengths=(1.0, 1.0, 1.0), device=None, group=None):
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if device is None:
            device = torch.cuda.current_device()
        mesh = build_box_mesh(ex, ey, ez, origin, lengths, periodic, deform)
        rank_of = partition_rcb(mesh, world)
        d = _box_desc(ex, ey, ez, degree, periodic, deform, origin, lengths)
        h = C.c_void_p()
        _check(lib.sbx_ctx_create_box_dist(C.byref(d), rank_of.ctypes.data, world, rank, device,
                                           C.byref(h)))
        size = lib.sbx_ctx_dist_blob_size(world)
        blob = (C.c_uint8 * size)()
        _check(lib.sbx_ctx_dist_blob(h, blob))
        blobs = [None] * world
        dist.all_gather_object(blobs, bytes(blob), group=group)
        allb = b"".join(blobs)
        buf = (C.c_uint8 * len(allb)).from_buffer_copy(allb)
        _check(lib.sbx_ctx_dist_connect(h, buf))
        ctx = cls(h, device)
        ctx.rank, ctx.world = rank, world
        ctx.rank_of = rank_of
        ids = np.zeros(ctx.elem_count, np.int64)
        _check(lib.sbx_ctx_local_elements(h, ids.ctypes.data))
        ctx.local_elements = ids
        ctx.global_elements = ex * ey * ez
        return ctx
