"""Host-side library logic on CPU (no GPU): the C ABI loads and exports every declared symbol;
the attention schedule covers every (sample, kv-head, m-tile, key block) exactly once and is
balanced."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rlhfspec_core.h")


@pytest.fixture(scope="module")
def core():
    from paper_2512_04752_b200 import build
    build.build(verbose=False)
    from paper_2512_04752_b200 import core as c
    return c


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(core):
    out = subprocess.run(["nm", "-D", "--defined-only", core.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    assert core.version().startswith("rlhfspec_core")


def _check_plan(core, P, T, Hq, Hkv, d=128, n=148):
    to = np.concatenate([[0], np.cumsum(T)]).astype(np.int32)
    pl = core.AttnPlan(P, to, Hq, Hkv, d, 64, num_ctas=n)
    cta, items = pl.schedule()
    info = pl.info()
    # static lists first; items past cta[-1] are the dynamic tail (pulled by CTAs that finished)
    assert cta[0] == 0 and cta[-1] <= len(items) and np.all(np.diff(cta) >= 0)
    g = Hq // Hkv
    # dual items (kernel RM = 4): every unit R = 32 with an even tile count -> an item covers
    # tiles (mt, mt + 1); tile 1's split parts follow tile 0's by item.pad
    dual = all(T[b] * g > 64 and ((T[b] * g + 127) // 128) % 2 == 0 for b in range(len(P)))
    cover = {}
    for b_, kvh, mt, b0, b1, part, R, unit, Pi, node0, Ti, pad in items:
        assert (Pi, node0, Ti) == (P[b_], to[b_], T[b_])       # lengths copied into the item
        assert (part < 0) == (unit < 0)
        for t in ((0, 1) if dual else (0,)):
            assert not dual or mt % 2 == 0
            cover.setdefault((b_, kvh, mt + t), []).append((b0, b1, part + t * pad if part >= 0 else -1))
    nsplit = 0
    for b in range(len(P)):
        nblk = (P[b] + T[b] + 63) // 64
        for kvh in range(Hkv):
            R = 16 if T[b] * g <= 64 else 32
            for mt in range((T[b] * g + 4 * R - 1) // (4 * R)):
                parts = sorted(cover.pop((b, kvh, mt)))
                assert parts[0][0] == 0 and parts[-1][1] == nblk
                assert all(x[1] == y[0] for x, y in zip(parts, parts[1:]))
                if len(parts) > 1:
                    nsplit += 1
                    assert all(p[2] >= 0 for p in parts)
                else:
                    assert parts[0][2] == -1
    assert not cover
    assert nsplit == info["num_split_units"]
    # per-item overhead the plan balances with (attention.cu: 2 blocks for the 16-warp kernel,
    # 6 for the 12-warp kernels, 1 for dual items)
    all16 = all(T[b] * g <= 64 for b in range(len(P)))
    ovh = 1 if dual else (2 if all16 else 6)
    loads = [sum(items[i, 4] - items[i, 3] + ovh for i in range(cta[c], cta[c + 1])) for c in range(len(cta) - 1)]
    return np.array(loads), info, pl


def test_plan_covers_and_balances_config2(core):
    loads, info, _ = _check_plan(core, np.full(64, 1024), np.full(64, 16), 32, 8)
    assert loads.max() <= 1.2 * loads.mean()


def test_plan_long_tail_and_gqa8(core):
    from synth import CONFIGS, draw_prefix_lengths
    rng = np.random.default_rng(0)
    P = draw_prefix_lengths(rng, CONFIGS["c3"])
    T = rng.integers(4, 65, size=len(P))
    loads, _, _ = _check_plan(core, P, T, 32, 8)
    assert loads.max() <= 1.05 * loads.mean()
    loads, _, _ = _check_plan(core, np.full(16, 8192), np.full(16, 64), 64, 8)
    assert loads.max() <= 1.05 * loads.mean()
    for n in (1, 3, 7):
        _check_plan(core, np.array([5000, 0, 20]), np.array([3, 37, 1]), 32, 8, n=n)


def test_plan_rejects_bad_trees(core):
    with pytest.raises(core.RSError):
        core.AttnPlan([10], [0, 65], 32, 8, 128, 64, 4)
    with pytest.raises(core.RSError):
        core.AttnPlan([10], [0, 0], 32, 8, 128, 64, 4)
    with pytest.raises(core.RSError):
        core.AttnPlan([10], [0, 4], 32, 8, 96, 64, 4)


def test_instance_migration_chunks_fit_staging(core):
    """Config 4 reallocation: a transfer's samples are cut into consecutive groups whose packed
    KV (LLM + SSM layers) fits the staging buffer; both ends derive the same groups."""
    from paper_2512_04752_b200.instance import GenerationInstance
    from paper_2512_04752_b200.realloc import SampleMeta
    inst = GenerationInstance.__new__(GenerationInstance)
    inst.L, inst.Hkv, inst.d = 32, 8, 128
    per_tok = 2 * 4 * 8 * 128 // 2 * 33            # bytes per token, 33 layers of K+V bf16
    rng = np.random.default_rng(0)
    metas = [SampleMeta(g, int(rng.integers(1, 3000)), 0.0) for g in range(40)]
    cap = 900 * 1024 * 1024
    groups = inst._chunks(metas, cap)
    assert [m.gid for g in groups for m in g] == list(range(40))       # order kept, nothing lost
    for g in groups:
        need = 2 * (core.kv_pack_elems(32, 8, 128, [m.seq_len for m in g]) +
                    core.kv_pack_elems(1, 8, 128, [m.seq_len for m in g]))
        assert need <= cap and need == sum(m.seq_len for m in g) * per_tok
    for a, b in zip(groups, groups[1:]):                               # greedy: next sample did not fit
        lens = [m.seq_len for m in a] + [b[0].seq_len]
        assert 2 * (core.kv_pack_elems(32, 8, 128, lens) + core.kv_pack_elems(1, 8, 128, lens)) > cap
    with pytest.raises(RuntimeError):
        inst._chunks([SampleMeta(0, 10 ** 6, 0.0)], cap)


def test_f1_f2_argument_validation(core):
    """The new entry points reject bad arguments before touching the device (CPU-only checks)."""
    import ctypes
    L = core._lib
    P = ctypes.c_void_p
    # rs_lm_head_argmax: Dm must be a positive multiple of 64; rows == 0 is a no-op
    assert L.rs_lm_head_argmax(P(16), P(16), 4, 100, 96, P(16), None, P(16), 64, None) == 1
    assert L.rs_lm_head_argmax(P(16), P(16), 4, 0, 128, P(16), None, P(16), 64, None) == 1
    assert L.rs_lm_head_argmax(None, None, 0, 100, 128, None, None, None, 0, None) == 0
    assert L.rs_lm_head_argmax(P(16), P(16), 4, 100, 128, None, None, P(16), 64, None) == 1
    assert L.rs_lm_head_argmax(P(16), P(16), 4, 100, 128, P(16), None, P(16), 8, None) == 11   # workspace
    assert core.lm_head_argmax_workspace_bytes(1000) == 8000
    # rs_tree_accept_greedy_tokens: B == 0 no-op, null pointers rejected
    assert L.rs_tree_accept_greedy_tokens(None, None, None, None, 0, None, None, None, None, None) == 0
    assert L.rs_tree_accept_greedy_tokens(None, None, None, None, 3, None, None, None, None, None) == 1
    # two-stage migration: a null communicator / descriptor is rejected
    assert L.rs_migrate_stage1(None, 0, 1, None, None, None, None, None, 1, None, 4, None, None, 0, None,
                               None) == 1
    assert L.rs_migrate_stage2(None, 0, 1, None, None, None, None, 1, None, 4, None, None, None, 0, None,
                               None, None) == 1


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the CPU oracle, runnable without a GPU) prints one JSON line
    with the base contract's keys plus impl / cpu_baseline / e2e (zero host<->device bytes)."""
    import json
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--config", "tiny",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("tiny")


def test_sampling_kernels_have_no_fused_multiply_add():
    """The bit-exact sampling arithmetic (exp_spec) is a fixed sequence of separately
    rounded fp32 multiplies and adds: the SASS of every acceptance kernel must contain no FFMA /
    FFMA2 (a contraction would change low bits and break parity with the C oracle)."""
    import shutil
    import subprocess
    from paper_2512_04752_b200 import build as B
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    obj = os.path.join(B.BUILD, "accept.cu.o")
    if not os.path.exists(obj):
        B.build(verbose=False)
    sass = subprocess.run([tool, "-sass", obj], capture_output=True, text=True, check=True).stdout
    funcs = [f for f in sass.split("Function : ")[1:] if "accept" in f.split("\n")[0] or "exp_spec" in f.split("\n")[0]]
    assert len(funcs) >= 6
    for f in funcs:
        assert "FFMA" not in f, f.split("\n")[0]


def test_accept_compact_argument_validation(core):
    """rs_tree_accept_compact rejects bad KV arguments before touching the device (CPU-only)."""
    import ctypes
    L = core._lib
    P = ctypes.c_void_p

    def call(B=3, L_=2, Hkv=8, d=128, ps=64, bt=P(16), pl=P(16), nl=P(16), kl=None, vl=None):
        k = (P * 2)(16, 16) if kl is None else kl
        v = (P * 2)(16, 16) if vl is None else vl
        return L.rs_tree_accept_compact(core.GREEDY, P(16), core.DTYPE_BF16, None, core.DTYPE_F32, None, P(16), P(16),
                                        P(16), P(16), B, 1000, 1.0, 0, 0, P(16), P(16), P(16), P(16), None, 0,
                                        k, v, L_, Hkv, d, ps, bt, 4, pl, nl, None, None)
    assert call(B=0) == 0                    # no samples: no-op
    assert call(L_=257) == 1                 # more layers than one launch's parameter block holds
    assert call(Hkv=0) == 1
    assert call(d=12) == 8                   # head_dim % 8 != 0: RS_ERR_UNSUPPORTED
    assert call(bt=None) == 1 and call(pl=None) == 1 and call(nl=None) == 1
    assert call(kl=(P * 2)(16, None)) == 1   # a null layer pointer
