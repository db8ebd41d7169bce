"""The fused edge passes (gather -> tcgen05 GEMM -> segmented per-destination
epilogue, csrc/tc.cuh + model.cu MsgSegProb / L7SegProb) against the unfused
kernel sequence (edge_a1 -> MsgProb -> segred forward, edge_bwd_prep
-> L7Prob -> segred backward; the fused passes are opt-in, HMTL_FUSE_EDGE=1), on
batches whose destinations
straddle 128-edge tiles and quadrants (mtl5 bench batch, max degree ~60) and
whose rows exceed a whole tile (cfg4 cells, degree > 128).  Same operations;
only a straddling destination's sum is associated per tile piece, so the two
agree to FP32 rounding (1e-6) and the fused path is bitwise reproducible."""
import os

import numpy as np
import pytest

import bench

import paper_2506_21788_b200 as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()
    if P.lib().hmtl_device_count() < 1:
        pytest.skip("no CUDA device")


def run(workload, fused, n_structs=None, steps=3, env=None):
    hyper = bench.WORKLOADS[workload]["hyper"]
    heads, batches, _ = bench.rank_batches(0, 1, nb=3, workload=workload)
    if n_structs:
        batches = [b.take(range(n_structs)) for b in batches]
    caps = P.Caps.for_samples(batches[0])
    for b in batches[1:]:
        caps = caps.union(P.Caps.for_samples(b))
    env = dict(env or {}, **({"HMTL_FUSE_EDGE": "1"} if fused else {}))
    os.environ.update(env)
    try:
        m = P.ModelT(P.ModelHyper(**hyper), 7, heads, caps=caps)
    finally:
        for k in env:
            os.environ.pop(k, None)
    cfg = P.TrainConfig(use_graph=True)
    losses = [m.train_step(batches[i % 3], cfg) for i in range(steps)]
    out = dict(losses=losses, agg=[m.debug("agg", l) for l in range(hyper["layers"])], g=m.grads().shared,
               p=m.shared_block(), pred=m.predictions().forces)
    m.close()
    return out


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(a), np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("workload,n", [("mtl5-weak", None), ("cfg4", 2), ("cfg2", None)])
def test_fused_edge_passes_match_unfused(workload, n):
    # one step: the same forward/backward at identical parameters (FP32 rounding only)
    a, b = run(workload, True, n, steps=1), run(workload, False, n, steps=1)
    np.testing.assert_allclose(a["losses"], b["losses"], rtol=1e-6)
    for x, y in zip(a["agg"], b["agg"]):
        assert rel(x, y) < 1e-6
    for k in ("g", "pred"):
        assert rel(a[k], b[k]) < 1e-5, k
    a, c = run(workload, True, n), run(workload, True, n)  # bitwise reproducible over steps
    assert a["losses"] == c["losses"]
    for k in ("g", "p", "pred"):
        assert np.array_equal(a[k], c[k]), k


@pytest.mark.parametrize("workload,n", [("mtl5-weak", None), ("cfg4", 2)])
def test_async_gather_producers_bit_identical(workload, n):
    """The cp.async gather producers (MsgAsyncProb / L7AsyncProb, tc.cuh kAsync: the
    default) compute the same operations as edge_a1 -> MsgProb and edge_bwd_prep ->
    L7Prob (HMTL_ASYNC_EDGE=0): every step bit-identical."""
    b = run(workload, False, n, env={"HMTL_ASYNC_FWD": "0", "HMTL_ASYNC_BWD": "0"})
    for env in ({"HMTL_ASYNC_FWD": "1", "HMTL_ASYNC_BWD": "1"}, {"HMTL_ASYNC_BWD": "1"}, {"HMTL_ASYNC_BWD": "2"}):
        a = run(workload, False, n, env=env)
        assert a["losses"] == b["losses"], env
        for x, y in zip(a["agg"], b["agg"]):
            assert np.array_equal(x, y), env
        for k in ("g", "p", "pred"):
            assert np.array_equal(a[k], b[k]), (env, k)


def test_force_output_layer_fused_into_dx_producer_bit_identical():
    """The force head's output-layer backward formed inside the dx GEMM's producer
    (FDxDsProb; its W_2/b_2 column sums on a side stream) == the separate elementwise
    pass (the default; the fused variant is opt-in, HMTL_FUSE_FORCE_OUT=1), every step bitwise."""
    a = run("mtl5-weak", False, env={"HMTL_FUSE_FORCE_OUT": "1"})
    b = run("mtl5-weak", False)
    assert a["losses"] == b["losses"]
    for k in ("g", "p", "pred"):
        assert np.array_equal(a[k], b[k]), k


def test_z1_only_storage_bit_identical():
    """The forward's edge pass storing z1 alone (consumers apply silu / silu'; opt-in
    HMTL_Z1_ONLY=1) == storing a1 and silu'(z1) (the default), every step bitwise."""
    a = run("mtl5-weak", False, env={"HMTL_Z1_ONLY": "1"})
    b = run("mtl5-weak", False)
    assert a["losses"] == b["losses"]
    for k in ("g", "p", "pred"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("cl", ["2", "4", "8"])
def test_cluster_split_k_reduce_matches(cl):
    """Weight-gradient split-K partials summed across a thread-block cluster through
    DSMEM (tc.cuh red_cluster_reduce; opt-in HMTL_RED_CLUSTER) == one partial per CTA
    reduced by split_reduce (the default): same sums in another order (FP32 rounding
    only), and bitwise reproducible over steps."""
    a = run("mtl5-weak", False, steps=1, env={"HMTL_RED_CLUSTER": cl})
    b = run("mtl5-weak", False, steps=1)
    np.testing.assert_allclose(a["losses"], b["losses"], rtol=1e-6)
    for k in ("g", "pred"):
        assert rel(a[k], b[k]) < 1e-5, k
    a, c = run("mtl5-weak", False, env={"HMTL_RED_CLUSTER": cl}), run("mtl5-weak", False, env={"HMTL_RED_CLUSTER": cl})
    assert a["losses"] == c["losses"]
    for k in ("g", "p", "pred"):
        assert np.array_equal(a[k], c[k]), k


def test_cta_pair_chain_matches():
    """Node-row chains as CTA-pair (cta_group::2, M = 256) kernels over pair-layout B
    images (opt-in HMTL_CHAIN_PAIR=1; chain.cuh pair_kernel) == the column-split
    cluster chains (the default): FP32 rounding only, bitwise reproducible."""
    a = run("mtl5-weak", False, steps=1, env={"HMTL_CHAIN_PAIR": "1"})
    b = run("mtl5-weak", False, steps=1)
    np.testing.assert_allclose(a["losses"], b["losses"], rtol=1e-6)
    for x, y in zip(a["agg"], b["agg"]):
        assert rel(x, y) < 1e-6
    for k in ("g", "pred"):
        assert rel(a[k], b[k]) < 1e-5, k
    a, c = run("mtl5-weak", False, env={"HMTL_CHAIN_PAIR": "1"}), run("mtl5-weak", False, env={"HMTL_CHAIN_PAIR": "1"})
    assert a["losses"] == c["losses"]
    for k in ("g", "p", "pred"):
        assert np.array_equal(a[k], c[k]), k


def test_l2_residency_knobs_bit_identical():
    """The persisting L2 window over the node tables (HMTL_L2_PERSIST_MB) and the
    chains' L2 prefetch (HMTL_CHAIN_PREFETCH) change only where bytes are cached:
    every step bitwise equal to the default."""
    a = run("mtl5-weak", False, env={"HMTL_L2_PERSIST_MB": "48", "HMTL_CHAIN_PREFETCH": "1"})
    b = run("mtl5-weak", False)
    assert a["losses"] == b["losses"]
    for k in ("g", "p", "pred"):
        assert np.array_equal(a[k], b[k]), k


def test_species_table_layer0_p_bit_identical():
    """Layer 0's P gathered from the per-species table T = embed [W1a | W1b] (built on the
    B-image side stream; the default) == the node-row P GEMM (HMTL_PTAB=0): the same
    tensor-core products per row, every step bitwise."""
    a = run("mtl5-weak", False)
    b = run("mtl5-weak", False, env={"HMTL_PTAB": "0"})
    assert a["losses"] == b["losses"]
    for k in ("g", "p", "pred"):
        assert np.array_equal(a[k], b[k]), k


def test_node_priority_and_wgrad_stream_bit_identical():
    """Scheduling knobs change only when kernels run: graph node priorities off
    (HMTL_NODE_PRIO=0) and the eW2 gradient on a third stream (HMTL_WGRAD3=2) give the
    default's bits on every step."""
    a = run("mtl5-weak", False)
    for env in ({"HMTL_NODE_PRIO": "0"}, {"HMTL_WGRAD3": "2"}):
        b = run("mtl5-weak", False, env=env)
        assert a["losses"] == b["losses"], env
        for k in ("g", "p", "pred"):
            assert np.array_equal(a[k], b[k]), (env, k)


def test_cta_pair_row_engine_bit_identical():
    """Row GEMMs over one segment as CTA pairs (opt-in HMTL_ROW_PAIR=1; tc.cuh kPair:
    tcgen05.mma.cta_group::2, M = 256, each CTA holding half of the resident B) == the
    single-CTA engine: the same per-row products in the same order, every step bitwise."""
    a = run("mtl5-weak", False, env={"HMTL_ROW_PAIR": "1"})
    b = run("mtl5-weak", False)
    assert a["losses"] == b["losses"]
    for k in ("g", "p", "pred"):
        assert np.array_equal(a[k], b[k]), k


def test_forward_chain_row_count_bit_identical():
    """Forward node chains in 64-row CTAs (M = 64 MMAs, twice the CTAs; the default) ==
    128-row CTAs (HMTL_CHAIN_M_FWD=128): the same per-row products, every step bitwise."""
    a = run("mtl5-weak", False)
    b = run("mtl5-weak", False, env={"HMTL_CHAIN_M_FWD": "128"})
    assert a["losses"] == b["losses"]
    for k in ("g", "p", "pred"):
        assert np.array_equal(a[k], b[k]), k
