"""Multi-process (gloo, world size 2, CPU) coverage of the row-partitioned path: every rank
plans its own rows (owned elements + ghosts) through the planning-only C ABI context; the
rank-0 check is that the concatenated rank patterns equal the world-1 pattern and the
oracle's, that each element is owned exactly once, and that the NCCL unique id bootstrap
(broadcast over the process group, as Assembler does) delivers identical bytes."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from fea_inputs import triangle_rule
        from fea_inputs.mesh import random_mesh_from_structured
        from paper_2204_03893_b200 import fea
        m = random_mesh_from_structured(7, p, seed=700 + p)
        ctx = fea.Context(device=-1, rank=rank, world=world)
        ctx.set_element(p, *triangle_rule(2 * p))
        ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
        ctx.build_pattern()
        rp, ci = ctx.get_pattern()
        mine = (ctx.row_begin, ctx.n_rows, rp, ci, ctx.stat(3), ctx.get_dof_perm())
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        try:
            uid = [fea.nccl_unique_id() if rank == 0 else None]
        except Exception:  # libnccl unavailable on this host: bootstrap bytes only
            uid = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        uids = [None] * world
        dist.all_gather_object(uids, uid[0])
        if rank == 0:
            q.put((allp, uids, m.n_dof, m.n_e))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("p", [1, 3])
def test_gloo_world2_row_partition(p):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    allp, uids, n_dof, n_e = q.get(timeout=180)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    import oracle
    from fea_inputs.mesh import random_mesh_from_structured
    from tests.helpers import lib_numbering
    m = random_mesh_from_structured(7, p, seed=700 + p)
    perm = allp[0][5]
    assert np.array_equal(perm, allp[1][5])  # same library numbering on every rank
    orp, oci = oracle.pattern(n_dof, lib_numbering(m, perm))
    rows, cols, nxt, owned = [0], [], 0, 0
    for (rb, nr, rp, ci, own, _) in allp:
        assert rb == nxt
        nxt += nr
        rows += list(rp[1:] + rows[-1])
        cols.append(ci)
        owned += own
    assert nxt == n_dof and owned == n_e
    assert np.array_equal(np.array(rows), orp) and np.array_equal(np.concatenate(cols), oci)
    assert uids[0] == uids[1] and len(uids[0]) == 128
