"""`h2ulv` alias (h2ulv_compat.install) and the host half of the batch
planner: CPU-only checks (no compute calls)."""
import sys

import numpy as np


def test_alias_maps_reference_module_names():
    from paper_2502_02395_b200 import h2ulv_compat
    pkg = h2ulv_compat.install()
    import h2ulv
    from h2ulv.dense_core import BlockOp, cholesky, id_basis, multiply, plan_batches, run_plan, tri_solve  # noqa: F401
    from h2ulv.h2_build import BuildConfig, build_basis_for_box, construct, h2_matvec  # noqa: F401
    from h2ulv.ulv_factor import (factor_diag, factorize, inject_couplings, merge_level,  # noqa: F401
                                  sparsify_diag, sparsify_off)
    from h2ulv.ulv_solve import backward_naive, backward_parallel, forward_naive, forward_parallel, solve  # noqa: F401
    assert h2ulv is pkg and sys.modules["h2ulv.ulv_factor"].__name__ == "paper_2502_02395_b200.ulv_factor"


def test_plan_batches_host_semantics():
    from paper_2502_02395_b200.dense_core import BlockOp, flop_count, plan_batches
    ops = [BlockOp(kind="multiply", dims=(m, m, m)) for m in (2, 7, 9, 13)]
    plan = plan_batches(ops, budget_blocks=2)
    assert [len(g.ops) for g in plan.groups] == [2, 2]
    assert all(g.padded_dims == (16, 16, 16) for g in plan.groups)
    assert plan.true_flops == sum(flop_count("multiply", (m, m, m)) for m in (2, 7, 9, 13))
    assert plan.padded_flops == 4 * flop_count("multiply", (16, 16, 16)) and plan.op_count == 4
    mixed = plan_batches([BlockOp(kind="cholesky", dims=(3,)), BlockOp(kind="tri_solve", dims=(5, 2))])
    assert sorted(g.kind for g in mixed.groups) == ["cholesky", "tri_solve"]
    assert [g.padded_dims for g in mixed.groups] == [(4,), (8, 4)]


def test_pad_for_cholesky():
    from paper_2502_02395_b200.dense_core import pad_for_cholesky
    p = pad_for_cholesky(np.array([[4.0, 1.0], [1.0, 3.0]]), 4)
    assert np.array_equal(p[2:, 2:], np.eye(2)) and np.array_equal(p[:2, 2:], np.zeros((2, 2)))
