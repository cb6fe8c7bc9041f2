"""Placement + cluster layer (include/psp/placement.hpp, include/psp/cluster.hpp):
the host mirrors against the reference build, the reference's own
test_cluster.cpp cases restated, and (GPU) routed_query / the sharded
RoutedOracle against the reference's routed_query and ClusterSim."""
import io
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1503_07192_b200 as P
from paper_1503_07192_b200 import cluster

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---- tests/test_cluster.cpp:19-38 -------------------------------------------
def test_round_robin_placement_stripes_components():
    pl = P.place_components(8, 3)
    assert pl.p == 3
    assert pl.owner.tolist() == [0, 1, 2, 0, 1, 2, 0, 1]
    assert pl.components_of == [[0, 3, 6], [1, 4, 7], [2, 5]]


def test_pairs_per_gpu_placement_blocks_components():
    assert P.place_components(8, 4, P.PAIRS_PER_GPU).owner.tolist() == [0, 0, 1, 1, 2, 2, 3, 3]
    assert P.place_components(7, 3, P.PAIRS_PER_GPU).owner.tolist() == [0, 0, 0, 1, 1, 2, 2]


def test_placement_validates_worker_counts():
    assert P.place_components(4, 1).owner.tolist() == [0, 0, 0, 0]
    with pytest.raises(ValueError):
        P.place_components(4, 0)
    with pytest.raises(ValueError):
        P.place_components(4, 5)
    with pytest.raises(ValueError):
        P.place_components(4, 2, "striped")


@pytest.mark.parametrize("policy", [P.ROUND_ROBIN, P.PAIRS_PER_GPU])
def test_placement_matches_reference(ref, policy):
    pol = 0 if policy == P.ROUND_ROBIN else 1
    for k in (1, 2, 5, 16, 17, 64, 1000):
        for p in (1, 2, 3, 4, 7, 8):
            if p > k:
                continue
            assert np.array_equal(P.place_components(k, p, policy).owner,
                                  ref.place_components(k, p, pol)), (k, p)


def test_ledger_accumulates_and_prints_csv():  # test_cluster.cpp:65-79
    ledger = P.TransferLedger()
    ledger.record(P.TransferRecord(1, 0, 1, 3, 24))
    ledger.record(P.TransferRecord(2, 1, 0, 5, 40))
    assert ledger.size() == 2
    assert ledger.total_entries() == 8
    assert ledger.total_bytes() == 64
    out = io.StringIO()
    ledger.write_csv(out)
    assert out.getvalue() == ("query_id,src_worker,dst_worker,entries,bytes\n"
                              "1,0,1,3,24\n"
                              "2,1,0,5,40\n")


def test_build_schedule_sums_component_costs_per_owner():  # test_cluster.cpp:137-152
    costs = [5, 5, 1, 1, 1, 1]
    rr = P.simulate_build_schedule(6, 2, costs)
    assert rr.worker_cost == [7, 7] and rr.makespan == 7 and rr.mean_load == 7
    blocks = P.simulate_build_schedule(6, 2, costs, P.PAIRS_PER_GPU)
    assert blocks.worker_cost == [11, 3] and blocks.makespan == 11 and blocks.mean_load == 7
    with pytest.raises(ValueError):
        P.simulate_build_schedule(6, 2, [1.0] * 5)


def test_build_schedule_matches_reference(ref):
    rng = np.random.default_rng(3)
    for k, p in ((16, 3), (64, 8), (100, 7)):
        costs = rng.uniform(0, 1e6, k)
        for pol, name in ((0, P.ROUND_ROBIN), (1, P.PAIRS_PER_GPU)):
            got = P.simulate_build_schedule(k, p, costs, name)
            wc, mk, ml = ref.simulate_build_schedule(k, p, costs, pol)
            assert got.worker_cost == wc and got.makespan == mk and got.mean_load == ml


def _expected_ledger(z, owner, v1, v2):
    """routed_query's transfer rule (cluster.cpp:77-84) restated on the
    fixture's reference partition: a record iff owner(C1) != owner(C2)."""
    # the fixture's assignment is indexed by original vertex id
    c1 = z["assignment"][v1.astype(np.int64)].astype(np.int64)
    c2 = z["assignment"][v2.astype(np.int64)].astype(np.int64)
    bo = z["boundary_offset"].astype(np.int64)
    b2 = bo[c2 + 1] - bo[c2]
    ex, co = owner[c1], owner[c2]
    idx = np.nonzero(ex != co)[0]
    return np.stack([idx, co[idx], ex[idx], b2[idx], 8 * b2[idx]], axis=1).astype(np.uint64)


def test_cluster_fixture_pins_transfer_rule(golden_cfg1):
    """The committed ClusterSim ledgers (tests/golden/ref_cluster_cfg1.npz,
    made by the reference) follow the transfer rule the GPU path returns."""
    zc = np.load(os.path.join(ROOT, "tests", "golden", "ref_cluster_cfg1.npz"))
    for p in (2, 4):
        for pol, name in ((0, P.ROUND_ROBIN), (1, P.PAIRS_PER_GPU)):
            owner = P.place_components(16, p, name).owner.astype(np.int64)
            want = zc[f"p{p}_pol{pol}_ledger"]
            assert np.array_equal(_expected_ledger(golden_cfg1, owner, zc["v1"], zc["v2"]), want)
            assert np.array_equal(zc[f"p{p}_pol{pol}_dist"], golden_cfg1["q_dist"][:len(zc["v1"])])


# ---- GPU: routed_query (cluster.cpp:49-74) ---------------------------------
@pytest.mark.gpu
def test_routed_query_ships_target_column(ref, ctx):  # test_cluster.cpp:41-63
    g = P.generate_grid(2, 3)
    o = P.build_oracle(g, 2, 1, 0, ctx=ctx)
    r = P.routed_query(o, P.place_components(2, 2), 0, 5, 17)
    assert r.result.distance == 3.0
    assert r.executed_on == 0 and r.column_owner == 1
    assert r.transfer == P.TransferRecord(17, 1, 0, 2, 16)
    assert r.result.transfer_entries == 2
    assert r.serial_cost == 2 * 2 + 2 + 2
    assert r.overlap_cost == 2 * 2 + 2
    local = P.routed_query(o, P.place_components(2, 1), 0, 5)
    assert local.transfer is None and local.result.transfer_entries == 0
    assert local.result.distance == 3.0 and local.serial_cost == 2 * 2 + 2


@pytest.mark.gpu
def test_routed_query_matches_reference(ref, ctx):
    rg = ref.generate("grid", 24, 24, (1.0, 9.0), 3)
    eu, ev, ew = rg.edges()
    g = P.Graph(rg.n, eu, ev, ew)
    o = P.build_oracle(g, 12, 2, 0, ctx=ctx)
    ro = rg.build_oracle(12, 2, 0)
    v1, v2 = P.random_pairs(g.n, 200, 9)
    for p, policy, pol in ((3, P.ROUND_ROBIN, 0), (4, P.PAIRS_PER_GPU, 1)):
        pl = P.place_components(12, p, policy)
        for i in range(len(v1)):
            got = P.routed_query(o, pl, int(v1[i]), int(v2[i]), i)
            want = ro.routed_query(p, int(v1[i]), int(v2[i]), i, pol)
            assert got.result.distance == want["distance"]
            assert got.result.minplus_ops == want["minplus_ops"]
            assert (got.result.boundary_size_1, got.result.boundary_size_2) == (want["b1"], want["b2"])
            assert got.result.same_component == bool(want["same_component"])
            assert got.result.transfer_entries == want["transfer_entries"]
            assert (got.executed_on, got.column_owner) == (want["executed_on"], want["column_owner"])
            assert (got.transfer is not None) == bool(want["has_transfer"])
            if got.transfer is not None:
                assert (got.transfer.src_worker, got.transfer.dst_worker, got.transfer.entries,
                        got.transfer.bytes) == (want["src_worker"], want["dst_worker"],
                                                want["entries"], want["bytes"])
            assert (got.overlap_cost, got.serial_cost) == (want["overlap_cost"], want["serial_cost"])


# ---- GPU: the sharded RoutedOracle ------------------------------------------
@pytest.mark.gpu
def test_routed_oracle_one_rank_matches_batch_query(ref, ctx):
    """p = 1 (test_cluster.cpp:125-135): one worker owns everything, so the
    routed batch equals batch_query and nothing crosses."""
    rg = ref.generate("tri", 30, 30, (0.25, 2.0), 1)
    eu, ev, ew = rg.edges()
    g = P.Graph(rg.n, eu, ev, ew)
    o = P.build_oracle(g, 20, 2, 0, ctx=ctx)
    v1, v2 = P.random_pairs(g.n, 20000, 4)
    want = o.batch_query(v1, v2)
    ro = P.RoutedOracle(o, P.place_components(o.k, 1))
    got, ex, co, ent = ro.run_batch(v1, v2, with_routing=True)
    assert np.array_equal(got, want)
    assert not ex.any() and not co.any() and not ent.any()
    assert ro.ledger().size() == 0
    assert ro.last_stats["executed_here"] == len(v1)
    assert ro.run_batch([], []).shape == (0,)
    with pytest.raises(ValueError):
        ro.run_batch([0, g.n], [1, 2])
    ro.close()


@pytest.mark.gpu
def test_routed_oracle_multi_rank():
    """2-4 ranks over NCCL + NVLink: distances bit-equal to the replicated
    oracle, ledger equal to the reference ClusterSim's (tools/routed_check.py)."""
    n = P._lib.lib().psp_gpu_device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={min(n, 4)}", "--master-addr=127.0.0.1",
                        "--master-port=29533", os.path.join(ROOT, "tools", "routed_check.py")],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "routed_check: ok" in r.stdout


@pytest.mark.gpu
def test_row_sharded_storage_full_size():
    """STORAGE_ROW_SHARDED at configs[1] size on 2-4 ranks: each rank keeps
    ~1/world of the boundary-graph table, RoutedOracle gathers its rows, and
    routed distances equal f64 Dijkstra (tools/row_storage_check.py)."""
    n = P._lib.lib().psp_gpu_device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={min(n, 4)}", "--master-addr=127.0.0.1",
                        "--master-port=29534", os.path.join(ROOT, "tools", "row_storage_check.py"),
                        "--config", "delaunay262k_k256"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "row_storage_check: ok" in r.stdout
    line = json.loads(next(x for x in r.stdout.splitlines() if x.startswith("{")))
    world = line["world"]
    for owned in line["owned_row_bytes_per_rank"]:
        assert owned <= line["table_bytes"] / world * 1.05


def test_set_boundary_storage_rejects_bad_values():
    # host-side argument check, no GPU needed: a NULL context is refused first
    L = P._lib.lib()
    assert L.psp_gpu_ctx_set_boundary_storage(None, P.STORAGE_ROW_SHARDED) == P._lib.PSP_EINVAL
