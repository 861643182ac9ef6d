"""The c3s workload's trees come from select_strategy (a0, host C++) run on candidate draft
trees: every verification tree is the root plus S(n) for the batch's single n (reading Z20),
which must be a connected, topologically ordered subtree of the candidates."""
import numpy as np

import bench
from oracle import strategy as OS
from synth import CONFIGS


def test_strategy_trees_are_connected_prefix_subtrees():
    from paper_2512_04752_b200 import core
    cfg = CONFIGS["c3s"]
    cfg = type(cfg)(**{**cfg.__dict__, "B": 24})
    st = bench.Strategy(cfg, core, "cpu", calibrate=False)   # prior F / t_sd: host-only, no GPU work
    cands, P, res, parents = st.cands, st.P, st.res, st.parents
    n = res["n"]
    ref = OS.select_strategy(cands, P, bench.STRATEGY_KX, bench.STRATEGY_KY,
                             OS.CostModel(**bench.STRATEGY_COST), n_min=3, n_max=63, patience=2)
    assert n == ref["n"] and 3 <= n <= 63
    for b, par in enumerate(parents):
        assert len(par) == n + 1 and par[0] == -1
        assert all(0 <= par[i] < i for i in range(1, n + 1))        # topological, rooted
        chosen = sorted(st.selected[b][:n])
        cp = cands[b][0]
        for c in chosen:                                            # S(n) closed under parent
            assert cp[c] < 0 or cp[c] in chosen
