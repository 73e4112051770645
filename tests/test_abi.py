"""C-ABI checks that need no GPU: the library loads, exports every symbol include/paradl.h
declares, struct layouts match, and host-side validation / sweep sizing behave."""
from __future__ import annotations

import os
import re
import subprocess

import pytest

from workloads import corpus
from workloads import models as M
from workloads import sweeps as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "paradl.h")


@pytest.fixture(scope="module")
def P():
    from paper_2104_09075_b200 import build
    build.build()
    import paper_2104_09075_b200 as P
    return P


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(paradl_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(P):
    names = declared_functions()
    assert len(names) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (paradl_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    from paper_2104_09075_b200 import _abi
    assert sorted(_abi.EXPORTS) == names


def test_library_is_sm100a(P):
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_sizes(P):
    from paper_2104_09075_b200 import _abi
    assert P.lib().paradl_struct_size(0) == 160
    for i, st in enumerate(_abi.STRUCTS):
        import ctypes
        assert P.lib().paradl_struct_size(i) == ctypes.sizeof(st)


@pytest.mark.parametrize("seed", range(20))
def test_sweep_size_matches_oracle(P, oracle_mod, seed):
    sw = corpus.random_sweep(seed)
    ctx = P.Context(-1)
    spec = ctx.prepare(sw)
    assert ctx.sweep_size(spec) == oracle_mod.OracleSweep(sw).size()


def test_named_config_sizes(P):
    expect = {1: 33, 2: 2_914_136_064, 3: 137_440_034_816, 4: 158_146_560, 5: 81_055_466_496}
    for i, n in expect.items():
        ctx = P.Context(-1)
        spec = ctx.prepare(W.CONFIGS[i]())
        assert ctx.sweep_size(spec) == n


def test_host_only_context_refuses_compute(P):
    ctx = P.Context(-1)
    spec = ctx.prepare(W.config1())
    with pytest.raises(P.ParadlError) as e:
        ctx.topk(spec, 4)
    assert e.value.status == -6   # ESTATE: no CPU fallback


def test_validation_errors(P):
    ctx = P.Context(-1)
    m = M.resnet(50)
    bad = M.resnet(50)
    bad.layers[3].x += 1
    with pytest.raises(P.ParadlError) as e:
        ctx.load_model(bad)
    assert e.value.status == -1 and "x != C*prod(X)" in str(e.value)
    bad = M.resnet(50)
    bad.layers[5].w += 7                      # not flagged FOLDED
    with pytest.raises(P.ParadlError):
        ctx.load_model(bad)
    ctx.load_model(m)
    s = W.two_tier_system()
    s.tiers = [W.Tier(8, 1e-6, 1e-9), W.Tier(8, 1e-6, 1e-9)]   # not strictly increasing
    with pytest.raises(P.ParadlError):
        ctx.set_system(s)
    s = W.two_tier_system(gamma=1.5)
    with pytest.raises(P.ParadlError):
        ctx.set_system(s)
    s = W.two_tier_system(delta=3)
    with pytest.raises(P.ParadlError):
        ctx.set_system(s)
    ctx.set_system(W.two_tier_system())
    from paper_2104_09075_b200 import Spec
    for sub in (W.SubSweep(W.SPATIAL, b=[1], dims=[(2, 2, 1, 1)], Ls=[3]),        # p1 != 1 for spatial
                W.SubSweep(W.SPATIAL, b=[1], dims=[(1, 2, 1, 1)]),                # no Ls list
                W.SubSweep(W.PIPELINE, b=[1]),                                    # no partition mode
                W.SubSweep(W.DATA, b=[1], part_mode=W.PART_COMB, s_max=2),        # partition on flat family
                W.SubSweep(W.PIPELINE, b=[1], part_mode=W.PART_COMB, s_min=1, s_max=17),
                W.SubSweep(W.PIPELINE, b=[1], part_mode=W.PART_MASK),            # G = 50 > 64? no: ok
                W.SubSweep(W.DATA, b=[]),
                W.SubSweep(W.DATA, b=[1], dims=[(0, 1, 1, 1)])):
        spec = Spec([sub], [0])
        if sub.part_mode == W.PART_MASK:
            assert ctx.sweep_size(spec) == 2 ** 49
            continue
        with pytest.raises(P.ParadlError):
            ctx.sweep_size(spec)
    # overflow proof: a batch so large that B * sum(FLOPs) could pass 2^62
    spec = Spec([W.SubSweep(W.DATA, b=[1 << 38], dims=[(1 << 20, 1, 1, 1)])], [0])
    with pytest.raises(P.ParadlError) as e:
        ctx.sweep_size(spec)
    assert e.value.status in (-1, -4)


def test_mask_mode_limit(P):
    ctx = P.Context(-1)
    ctx.load_model(M.resnet(152))
    ctx.set_system(W.two_tier_system())
    from paper_2104_09075_b200 import Spec
    with pytest.raises(P.ParadlError):
        ctx.sweep_size(Spec([W.SubSweep(W.PIPELINE, b=[1], part_mode=W.PART_MASK)], [0]))
