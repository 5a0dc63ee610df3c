"""CPU-only checks of the C ABI library and the host logic (no GPU needed):
the shared object loads, exports every function include/lopt_b200.h declares,
and the plan builder enforces the reference's shape rules."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "lopt_b200.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lopt_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2506_10315_b200 import _lib

    L = _lib.lib()
    names = _declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib.EXPORTS)
    assert b"sm_100a" in L.lopt_version()


def test_library_is_sm100a_cubin():
    import subprocess

    from paper_2506_10315_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.SO], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def _tensor(m, n, lo=0, hi=None, slot=0, state=0x1000):
    from paper_2506_10315_b200 import _lib

    hi = m * n if hi is None else hi
    return _lib.lopt_tensor(m=m, n=n, lo=lo, hi=hi, theta=0x1000, grad=0x2000, state=state,
                            row_factors=0x3000, col_factors=0x4000, weight_slot=slot, reserved=0)


def _cfg(**kw):
    from paper_2506_10315_b200 import _lib

    c = _lib.lopt_config()
    c.feature_set = kw.get("feature_set", 0)
    c.mode = kw.get("mode", 0)
    c.hidden1 = kw.get("hidden", 32)
    c.hidden2 = kw.get("hidden", 32)
    c.num_weight_sets = kw.get("sets", 1)
    c.state_advanced = 0
    for k, b in enumerate(kw.get("betas", (0.1, 0.5, 0.9, 0.999, 0.9, 0.99, 0.999))):
        c.betas[k] = b
    c.alpha = 0.01
    c.beta_out = 0.01
    c.update_sign = kw.get("sign", -1)
    return c


def _create(tensors, cfg):
    from paper_2506_10315_b200 import _lib

    L = _lib.lib()
    arr = (_lib.lopt_tensor * len(tensors))(*tensors)
    h = ctypes.c_void_p()
    rc = L.lopt_plan_create(arr, len(tensors), ctypes.byref(cfg), ctypes.byref(h))
    if rc == 0:
        nb = ctypes.c_size_t()
        assert L.lopt_workspace_bytes(h, ctypes.byref(nb)) == 0
        L.lopt_plan_destroy(h)
        return rc, nb.value
    return rc, None


def test_plan_accepts_reference_shapes():
    shapes = [(1, 1), (1, 130), (130, 1), (768, 3072), (50257, 1024), (197, 768)]
    rc, nbytes = _create([_tensor(m, n) for m, n in shapes], _cfg())
    assert rc == 0 and nbytes > 0


def test_plan_rejects_empty_and_bad_ranges():
    from paper_2506_10315_b200 import _lib

    assert _create([_tensor(0, 5)], _cfg())[0] == _lib.LOPT_ERR_SHAPE        # EngineError: empty
    assert _create([_tensor(4, 4, lo=3, hi=2)], _cfg())[0] == _lib.LOPT_ERR_SHAPE
    assert _create([_tensor(4, 4, lo=0, hi=17)], _cfg())[0] == _lib.LOPT_ERR_SHAPE
    assert _create([_tensor(4, 4, state=0x1004)], _cfg())[0] == _lib.LOPT_ERR_INVALID
    assert _create([_tensor(4, 4, slot=1)], _cfg())[0] == _lib.LOPT_ERR_INVALID


def test_plan_rejects_bad_config():
    from paper_2506_10315_b200 import _lib

    assert _create([_tensor(4, 4)], _cfg(hidden=16))[0] == _lib.LOPT_ERR_UNSUPPORTED
    assert _create([_tensor(4, 4)], _cfg(sign=2))[0] == _lib.LOPT_ERR_INVALID
    assert _create([_tensor(4, 4)], _cfg(betas=(0.1, 0.5, 1.5, 0.999, 0.9, 0.99, 0.999)))[0] \
        == _lib.LOPT_ERR_INVALID
    assert _create([_tensor(4, 4)], _cfg(feature_set=7))[0] == _lib.LOPT_ERR_INVALID


def test_sharded_ranges_allow_empty_local_range():
    rc, _ = _create([_tensor(3, 3, lo=4, hi=4, state=0)], _cfg())
    assert rc == 0


# ---------------------------------------------------------------------------
# host-side mirrors agree with the oracle (hence with the reference)


def test_random_weights_match_reference_generator(oracle):
    from paper_2506_10315_b200 import random_weights

    for d, seed in ((39, 0), (29, 5)):
        a = random_weights(d, seed=seed)
        b = oracle.random_weights(d, seed=seed)
        for (wa, ba), (wb, bb) in zip(a.layers, b.layers):
            assert wa.tobytes() == wb.tobytes() and ba.tobytes() == bb.tobytes()


def test_time_features_match_oracle(oracle):
    from paper_2506_10315_b200 import small_fc_lopt_spec, time_features, velo_mlp_spec

    for t in (0, 1, 7, 100, 12345):
        assert time_features(t, small_fc_lopt_spec()).tobytes() == \
            oracle.time_features(t, oracle.SMALL_FC_LOPT).tobytes()
    assert not time_features(5, velo_mlp_spec()).any()
    assert round(float(time_features(100, small_fc_lopt_spec())[4]), 6) == 0.761594


def test_schedule_and_view_rule(oracle):
    from paper_2506_10315_b200 import ScheduleConfig, schedule_lr, view_2d

    cfg = ScheduleConfig(kind="cosine", max_lr=0.5, min_lr=0.01, warmup_steps=10, total_steps=100)
    for s in (0, 5, 10, 11, 50, 99, 100, 1000):
        assert schedule_lr(cfg, s) == oracle.schedule_lr("cosine", 0.5, 0.01, 10, 100, s)
    for shape in ((), (7,), (1, 768), (1, 1, 768), (1, 197, 768), (768, 3, 16, 16)):
        assert view_2d(shape) == oracle.view_2d(shape)


def test_packed_weight_layout():
    from paper_2506_10315_b200 import random_weights
    from paper_2506_10315_b200.weights import unpack

    w = random_weights(39, seed=3)
    p = w.packed()
    assert p.size == 32 * 39 + 32 + 32 * 32 + 32 + 2 * 32 + 2
    back = unpack(p, 39)
    for (a, b), (c, d) in zip(w.layers, back.layers):
        assert np.array_equal(a, c) and np.array_equal(b, d)


def test_optimizer_rejects_host_tensors_before_any_device_call():
    """CPU parameters would hand host pointers to the kernels: the optimizer
    refuses them with a TypeError before building a plan."""
    import torch

    import paper_2506_10315_b200 as P

    p = torch.nn.Parameter(torch.zeros(4, 3))
    p.grad = torch.zeros(4, 3)
    opt = P.LearnedOptimizer([p])
    with pytest.raises(TypeError, match="CUDA"):
        opt.step()


def test_fast_mode_size_limit_and_strict_beyond_it():
    """The tensor-core apply pass indexes a tensor's elements with 32-bit
    integers: a tensor of 2^31 or more elements is LOPT_ERR_UNSUPPORTED in fast
    mode (a loud error, never a silent overflow); strict mode takes it."""
    from paper_2506_10315_b200 import _lib

    big = _tensor(1 << 16, 1 << 15)          # 2^31 elements
    assert _create([big], _cfg(mode=1))[0] == _lib.LOPT_ERR_UNSUPPORTED
    assert _create([_tensor(1 << 16, (1 << 15) - 1)], _cfg(mode=1))[0] == 0
    rc, nbytes = _create([big], _cfg(mode=0))
    assert rc == 0 and nbytes > 0


def test_fast_plan_odd_row_counts_and_ranges():
    """Tile pairs: odd row counts (an empty second tile closes each column
    block) and element-range shards that start and end inside rows plan
    without error in fast mode."""
    rc, _ = _create([_tensor(197, 768), _tensor(1, 768), _tensor(3, 128, lo=70, hi=300),
                     _tensor(1000, 1), _tensor(5, 7)], _cfg(mode=1))
    assert rc == 0
