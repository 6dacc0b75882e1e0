"""World-size-2 runs of the row-partitioned GPU path on ONE GPU, every rank checked against the
ORACLE (VERDICT r1 "What's missing" 1 / "Next round" 4).  Two processes (torch.multiprocessing,
gloo process group on CPU) share cuda:0; the exchange of u between them goes over gloo on host
buffers, so no kernel of one rank waits on the other's.  Covered, for P1-P4 configs:

* fea_reassemble through the library's own exchange path with a HOST transport
  (fea_set_host_transport: pack kernel -> D2H -> gloo allgather -> H2D -> unpack kernel) in both
  exchange modes (interface-only / full vector) and with the overlap on (interior blocks on the
  ctx stream while the exchange runs on the second stream, boundary blocks after the halo event)
  and off -- the code path NCCL takes, minus the NCCL call itself;
* the caller-transport split: fea_exchange_pack -> gloo all_gather -> fea_exchange_unpack ->
  fea_assemble.

Each rank compares its rows [row_begin, row_begin + n_rows) with the oracle's rows in library
numbering: pattern bit-exact, values within the north-star tolerance."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, N, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        from fea_inputs import CONFIGS, MASS, STIFF, make_workload, scaled
        from paper_2204_03893_b200.fea import Context
        from tests.helpers import maxabs_rel, oracle_for
        cfg = scaled(CONFIGS[name], N)
        wl = make_workload(cfg)
        m = wl.mesh
        mc, cc = cfg.coef_m, cfg.coef_c
        dev = "cuda:0"

        def gloo_allgather(send, recv):
            n = send.shape[0]
            outs = [torch.from_numpy(recv[k * n:(k + 1) * n]) for k in range(world)]
            dist.all_gather(outs, torch.from_numpy(send.copy()))

        def make(tuning):
            ctx = Context(device=0, rank=rank, world=world)
            ctx.set_element(cfg.p, wl.q_xy, wl.q_w)
            ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, reorder=cfg.reorder)
            ctx.set_tuning(4, cfg.which)
            for k, v in tuning.items():
                ctx.set_tuning(k, v)
            ctx.build_pattern()
            ctx.set_coefficient(MASS, *mc)
            ctx.set_coefficient(STIFF, *cc)
            return ctx

        ref = None
        for mode, tuning in (("lib-iface-overlap", {}), ("lib-iface-serial", {7: 0}), ("lib-full", {5: 1}),
                             ("caller-transport", {})):
            ctx = make(tuning)
            perm = ctx.get_dof_perm()
            R0, nr, nnz = ctx.row_begin, ctx.n_rows, ctx.nnz
            if ref is None:
                ref = oracle_for(m, wl.q_xy, wl.q_w, wl.u0, perm, mc, cc, cfg.which, r0=R0, r1=R0 + nr)
            u_lib = torch.tensor(wl.u0[perm], dtype=torch.float64, device=dev)
            u_own = u_lib[R0:R0 + nr].contiguous()
            M = torch.full((max(nnz, 1),), np.nan, dtype=torch.float64, device=dev) if cfg.which & MASS else None
            K = torch.full((max(nnz, 1),), np.nan, dtype=torch.float64, device=dev) if cfg.which & STIFF else None
            if mode.startswith("lib"):
                ctx.set_host_transport(gloo_allgather)
                for _ in range(2):  # a second call reuses the pinned buffers and the plan
                    ctx.reassemble(u_own, M, K)
                ctx.sync()
            else:
                maxI = ctx.stat(14)
                send = torch.zeros(max(maxI, 1), dtype=torch.float64, device=dev)
                ctx.exchange_pack(u_own, send)
                ctx.sync()
                recv_h = np.zeros(world * max(maxI, 1))
                if maxI:
                    gloo_allgather(send[:maxI].cpu().numpy(), recv_h[:world * maxI])
                recv = torch.tensor(recv_h, device=dev)
                u_full = torch.full((m.n_dof,), np.nan, dtype=torch.float64, device=dev)  # only what is read
                ctx.exchange_unpack(u_own, recv, u_full)
                ctx.assemble(u_full, M, K)
                ctx.sync()
            rp, ci = ctx.get_pattern()
            res = {"mode": mode, "rank": rank, "pattern": bool(np.array_equal(rp, ref.row_ptr)
                                                               and np.array_equal(ci, ref.col_idx)),
                   "interior": ctx.stat(15), "blocks": ctx.stat(1)}
            for key, got, want in (("M", M, ref.M), ("K", K, ref.K)):
                if got is not None:
                    g = got[:nnz].cpu().numpy()
                    res[key] = maxabs_rel(g, want) if np.isfinite(g).all() else float("inf")
            out.append(res)
            ctx.close()
    except Exception as e:  # reported to the test process
        import traceback
        out.append({"error": f"rank {rank}: {e!r}\n{traceback.format_exc()}"})
    finally:
        q.put(out)
        dist.destroy_process_group()


@pytest.mark.parametrize("name,N", [("C1", 16), ("C2", 20), ("C3", 12), ("C4", 40), ("C5", 8)])
def test_world2_gloo_exchange_vs_oracle(name, N):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, N, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
    flat = [r for rs in results for r in rs]
    errs = [r["error"] for r in flat if "error" in r]
    assert not errs, errs[0]
    assert len(flat) == 4 * world
    for r in flat:
        assert r["pattern"], r
        for key in ("M", "K"):
            if key in r:
                assert r[key] <= TOL, r
    for pr in procs:
        assert pr.exitcode == 0
