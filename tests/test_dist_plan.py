"""Multi-GPU host logic on CPU: world_size 2 and 3 over torch.distributed/gloo.

Every rank builds its exchange plan (libsbx.so host code, no GPU), performs
the distributed gather-scatter exactly as the device path does (pack raw copy
values -> exchange -> interface groups summed in canonical order -> local
boundary groups) with gloo point-to-point messages standing in for the
NVLink peer stores, and checks the result is BITWISE the single-process
reference gs_sum (oracle) restricted to its elements.  Also checks the
multiplicity / mask / 27-neighbourhood tables against the global mesh.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

CASES = [
    dict(ex=6, ey=5, ez=4, N=3, per=(False, False, False), deform=0.05),
    dict(ex=4, ey=4, ez=6, N=5, per=(True, False, True), deform=0.0),
    dict(ex=8, ey=3, ez=3, N=2, per=(False, True, False), deform=0.03),
]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2109_03592_b200 as sb
        from oracle import oracle as O
        from paper_2109_03592_b200 import dist as sd

        for c in CASES:
            ex, ey, ez, N = c["ex"], c["ey"], c["ez"], c["N"]
            mesh = sb.build_box_mesh(ex, ey, ez, periodic=c["per"], deform=c["deform"])
            rank_of = sb.partition_rcb(mesh, world)
            P = sd.plan(ex, ey, ez, N, rank_of, world, rank, c["per"])
            n3 = (N + 1) ** 3
            assert np.array_equal(P["loc_elems"], np.nonzero(rank_of == rank)[0])
            G = O.Problem(ex, ey, ez, N, periodic=c["per"], corners=mesh.corners)
            f = O.fill_uniform(1234, G.nodes_count)
            ref = f.copy()
            G.gs_sum_inplace(ref)
            lnodes = (P["loc_elems"][:, None] * n3 + np.arange(n3)[None, :]).ravel()
            NL = P["nodes_local"]
            assert NL == lnodes.size
            assert np.array_equal(P["inv_mult"], G.inv_mult[lnodes])
            assert np.array_equal(P["mask"], G.mask[lnodes])
            raw = f[lnodes].copy()
            w = raw.copy()
            # exchange of raw copy values (gloo p2p in place of NVLink stores)
            reqs, recv = [], np.zeros(max(P["recv_total"], 1))
            send_off = np.concatenate([[0], np.cumsum(P["send_count"])])
            rbufs = []
            for qi, nb in enumerate(P["nbr"]):
                sbuf = torch.from_numpy(raw[P["send_idx"][send_off[qi]:send_off[qi + 1]]].copy())
                rbuf = torch.zeros(int(P["recv_count"][qi]), dtype=torch.float64)
                reqs.append(dist.isend(sbuf, int(nb)))
                reqs.append(dist.irecv(rbuf, int(nb)))
                rbufs.append((qi, rbuf))
            for r in reqs:
                r.wait()
            for qi, rbuf in rbufs:
                b0 = int(P["recv_base"][qi])
                recv[b0:b0 + rbuf.numel()] = rbuf.numpy()
            # interface groups, canonical order
            for g in range(len(P["if_off"]) - 1):
                lo, hi = P["if_off"][g], P["if_off"][g + 1]
                s = 0.0
                for code in P["if_code"][lo:hi]:
                    s += recv[code - NL] if code >= NL else raw[code if code >= 0 else ~code]
                for code in P["if_code"][lo:hi]:
                    if code < NL:
                        w[code if code >= 0 else ~code] = s
            # local boundary groups (gather.cpp:85-98 semantics)
            for g in range(len(P["b_off"]) - 1):
                lo, hi = P["b_off"][g], P["b_off"][g + 1]
                if hi - lo == 1:
                    continue
                idx = [a if a >= 0 else ~a for a in P["b_idx"][lo:hi]]
                s = 0.0
                for a in idx:
                    s += raw[a]
                for a in idx:
                    w[a] = s
            assert np.array_equal(w, ref[lnodes]), "distributed gs differs from gs_sum"
            # 27-neighbourhood
            E = ex * ey * ez
            for le in range(0, len(P["loc_elems"]), 7):
                e = int(P["loc_elems"][le])
                cx, cy, cz = e % ex, (e // ex) % ey, e // (ex * ey)
                for dz in (-1, 0, 1):
                    for dy in (-1, 0, 1):
                        for dx in (-1, 0, 1):
                            cc, inside = [cx + dx, cy + dy, cz + dz], True
                            for d, cnt in enumerate((ex, ey, ez)):
                                if not 0 <= cc[d] < cnt:
                                    if c["per"][d]:
                                        cc[d] %= cnt
                                    else:
                                        inside = False
                            code = P["nbr27"][le * 27 + (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)]
                            if not inside:
                                assert code == -1
                            else:
                                ge = cc[0] + ex * (cc[1] + ey * cc[2])
                                assert ge < E
                                if rank_of[ge] == rank:
                                    assert P["loc_elems"][code] == ge
                                else:
                                    assert code == -2
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_distributed_gs_plan_bitwise(world):
    ctx = mp.get_context("spawn")
    for _attempt in range(3):  # (a rendezvous port taken meanwhile: pick another)
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        results = [q.get(timeout=300) for _ in range(world)]
        for p in procs:
            p.join(timeout=60)
        if not any("address already in use" in msg.lower() or "EADDRINUSE" in msg
                   for _, msg in results):
            break
    for rank, msg in results:
        assert msg == "ok", f"rank {rank}:\n{msg}"


def test_plan_single_rank_has_no_interface():
    import paper_2109_03592_b200 as sb
    from paper_2109_03592_b200 import dist as sd

    mesh = sb.build_box_mesh(3, 3, 3)
    P = sd.plan(3, 3, 3, 3, np.zeros(27, np.int32), 1, 0)
    assert len(P["nbr"]) == 0 and len(P["if_off"]) == 1 and P["recv_total"] == 0
    assert (P["nbr27"] != -2).all()
