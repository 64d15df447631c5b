"""World-size-2 (gloo, CPU) test of the multi-GPU data flow.

Each rank takes its share of the plan from the C++ layout layer
(pdd_rank_layout: subdomain d on rank floor(d*world/D), local pairs, NCCL
exchange schedule), runs one OD²P iteration on its own subdomains with the
oracle's arithmetic, exchanges s = pi u + Lambda over the cut pairs with
send/recv exactly as csrc/common.cuh consensus() does with NCCL, and reduces the
per-subdomain R-factor / RE partials through a single-contributor D-vector
all-reduce.  The result must equal the single-process oracle iteration.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(kind):
    from oracle import od2p as O
    from tests.golden import cases

    N, s, step = 96, 32, 8
    probe = cases.gaussian_probe(s, s / 4)
    g = O.make_raster_scan(N, N, s, step)
    f = O.intensity(O.forward(probe, cases.smooth_object(N, 7), g))
    if kind == "grid":
        return N, s, step, f, probe, ("grid", 2, 2)
    return N, s, step, f, probe, ("stripes", 3, "auto")


def _worker(rank, world, port, kind, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import od2p as O
        import paper_2011_00162_b200 as P
        from paper_2011_00162_b200 import dist as pdist

        N, s, step, f, probe, pk = _problem(kind)
        gp = P.make_raster_scan(N, N, s, step)
        plan = P.plan_grid(gp, pk[1], pk[2]) if pk[0] == "grid" else P.plan_stripes(gp, pk[1], pk[2])
        go = O.make_raster_scan(N, N, s, step)
        oplan = O.plan_grid(go, pk[1], pk[2]) if pk[0] == "grid" else O.plan_stripes(go, pk[1], pk[2])
        lay = pdist.rank_layout(plan, rank, world)
        D = plan.D
        assert all(int(d * world // D) == rank for d in lay.local_subs)

        # global oracle state after init (every rank can build it; only local parts are used)
        sol = O.NonblindSolver(oplan, f, probe, O.NonblindConfig())
        st = sol.init_state()
        au = [z.copy() for z in st.z]
        cfg = sol.config
        mine = set(lay.local_subs)
        # z / Gamma for local subdomains
        for d in mine:
            y = st.gamma[d] + au[d]
            st.z[d] = O.pixel_prox(y, sol.frames[d], cfg.eta, cfg.epsilon)
            st.gamma[d] = y - st.z[d]
        # s = pi u + Lambda for local sides, exchanged per the C++ schedule
        svals = {}
        for lp, p in enumerate(lay.local_pairs):
            ov = oplan.overlaps[p]
            for side, d in enumerate((ov.d1, ov.d2)):
                if d in mine:
                    other = ov.d2 if side == 0 else ov.d1
                    svals[(p, side)] = O.restrict_overlap(st.u[d], oplan, d, other) + st.lam[p][side]
        reqs = []
        recvbufs = {}
        for lp, peer, my_side in lay.exchange:
            p = lay.local_pairs[lp]
            send = torch.from_numpy(np.ascontiguousarray(svals[(p, my_side)]).view(np.float64).copy())
            recv = torch.empty_like(send)
            recvbufs[(p, 1 - my_side)] = recv
            reqs.append(dist.isend(send, peer))
            reqs.append(dist.irecv(recv, peer))
        for r in reqs:
            r.wait()
        for (p, side), t in recvbufs.items():
            svals[(p, side)] = t.numpy().view(np.complex128).reshape(svals[(p, 1 - side)].shape)
        for p in lay.local_pairs:
            st.v[p] = 0.5 * (svals[(p, 0)] + svals[(p, 1)])
        # u and Lambda updates for local subdomains / sides; RE partials
        part = np.zeros(3 * D)
        uprev = [u.copy() for u in st.u]
        for d in mine:
            lg = oplan.local_geometries[d]
            num = O.adjoint(probe, st.z[d] - st.gamma[d], lg) * cfg.eta
            num = O._consensus_terms(oplan, d, num, st, cfg.r)
            st.u[d] = np.where(sol.pin[d], 1.0 + 0j, num / sol.denom[d])
            for p in oplan.pairs_of(d):
                side = 0 if oplan.overlaps[p].d1 == d else 1
                other = oplan.overlaps[p].d2 if side == 0 else oplan.overlaps[p].d1
                st.lam[p][side] = st.lam[p][side] + (O.restrict_overlap(st.u[d], oplan, d, other) - st.v[p])
            dd = st.u[d] - uprev[d]
            part[D + d] = float(np.sum(np.abs(dd) ** 2))
            part[2 * D + d] = float(np.sum(np.abs(st.u[d]) ** 2))
            aud = O.forward(probe, st.u[d], lg)
            part[d] = float(np.sum(np.abs(np.abs(aud) - sol.sqrt_f[d])))
        t = torch.from_numpy(part)
        dist.all_reduce(t)  # single contributor per entry: exact
        part = t.numpy()
        rf = sum(part[d] for d in range(D)) / sol.sqrt_f_l1
        re = max(np.sqrt(part[D + d]) / np.sqrt(part[2 * D + d]) for d in range(D))
        q.put((rank, {d: st.u[d] for d in mine}, {p: st.v[p] for p in lay.local_pairs},
               {(p, sd): st.lam[p][sd] for p in lay.local_pairs for sd in (0, 1)
                if (oplan.overlaps[p].d1 if sd == 0 else oplan.overlaps[p].d2) in mine}, rf, re))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["stripes", "grid"])
def test_two_rank_iteration_equals_single_process(kind):
    sys.path.insert(0, ROOT)
    from oracle import od2p as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process oracle iteration
    N, s, step, f, probe, pk = _problem(kind)
    g = O.make_raster_scan(N, N, s, step)
    oplan = O.plan_grid(g, pk[1], pk[2]) if pk[0] == "grid" else O.plan_stripes(g, pk[1], pk[2])
    sol = O.NonblindSolver(oplan, f, probe, O.NonblindConfig())
    st = sol.init_state()
    au = [z.copy() for z in st.z]
    u0 = [u.copy() for u in st.u]
    sol.step(st, au)
    rf = sol.r_factor_of(au)
    re = O._relative_error_solver(st.u, u0)
    seen_u, seen_l = set(), set()
    for rank, us, vs, lams, rrf, rre in results:
        for d, u in us.items():
            assert np.max(np.abs(u - st.u[d])) < 1e-12 * np.max(np.abs(st.u[d]))
            seen_u.add(d)
        for p, v in vs.items():
            assert np.max(np.abs(v - st.v[p])) < 1e-12
        for (p, sd), lam in lams.items():
            assert np.max(np.abs(lam - st.lam[p][sd])) < 1e-12
            seen_l.add((p, sd))
        assert abs(rrf - rf) < 1e-12 * rf and abs(rre - re) < 1e-12 * re
    assert seen_u == set(range(oplan.D))
    assert len(seen_l) == 2 * len(oplan.overlaps)


def _id_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import bench

    d = bench.init_dist(world)
    try:
        q.put((rank, bench.fresh_nccl_id(d, rank, world), bench.fresh_nccl_id(d, rank, world)))
    finally:
        d.destroy_process_group()


def test_bench_draws_a_fresh_nccl_id_per_communicator():
    """bench.py builds two solvers per rank (timed loop, then e2e); an NCCL
    unique id bootstraps one communicator only, so each gets its own id, the
    same on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, a0, b0), (_, a1, b1) = res
    assert len(a0) == 128 and a0 == a1 and b0 == b1 and a0 != b0
