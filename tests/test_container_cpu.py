"""PYLO container / checkpoint interop on the host (no GPU): files written by
the reference (tests/golden/ref_*.pylo, made by gen_golden.py) are read
bit-exactly and re-written byte for byte."""

import os
import shutil

import numpy as np
import pytest

from conftest import ROOT

GOLD = os.path.join(ROOT, "tests", "golden")


def _C():
    from paper_2506_10315_b200 import container
    return container


@pytest.mark.parametrize("name", ["ref_misc", "ref_weights_small_const", "ref_weights_velo_cos_wd",
                                  "ref_ckpt_small_const", "ref_ckpt_velo_cos_wd"])
def test_reference_files_roundtrip_bytes(tmp_path, name):
    C = _C()
    src = os.path.join(GOLD, name + ".pylo")
    entries, meta = C.file_load(src)
    out = tmp_path / "again.pylo"
    C.file_save(entries, meta, out)
    assert out.read_bytes() == open(src, "rb").read()


def test_misc_entries():
    C = _C()
    e, meta = C.file_load(os.path.join(GOLD, "ref_misc.pylo"))
    assert e["a"].dtype == np.float32 and e["a"].shape == (2, 3)
    assert e["b"].shape == () and float(e["b"]) == 3.5 and e["b"].dtype == np.float64
    assert e["c"].dtype == np.int64 and e["c"].tolist() == [0, 1, 2, 3, 4]
    assert e["d"].shape == (0, 4)
    assert meta == {"kind": "misc", "note": "unicode é"}


def test_typed_errors(tmp_path):
    C = _C()
    src = open(os.path.join(GOLD, "ref_misc.pylo"), "rb").read()
    cases = {
        "magic": (b"XXXX" + src[4:], C.MalformedHeaderError),
        "version": (src[:4] + (2).to_bytes(4, "little") + src[8:], C.VersionMismatchError),
        "short": (src[:10], C.TruncatedFileError),
        "payload": (src[:-8], C.TruncatedFileError),
    }
    for k, (blob, err) in cases.items():
        p = tmp_path / f"{k}.pylo"
        p.write_bytes(blob)
        with pytest.raises(err):
            C.file_load(p)


@pytest.mark.parametrize("run,fs,seed", [("small_const", "small_fc_lopt", 3),
                                         ("velo_cos_wd", "velo_mlp", 4)])
def test_reference_weights_are_random_weights(run, fs, seed, oracle):
    C = _C()
    w, got_fs = C.load_weights(os.path.join(GOLD, f"ref_weights_{run}.pylo"), expect=fs)
    assert got_fs == fs
    ref = oracle.random_weights(39 if fs == "small_fc_lopt" else 29, seed=seed)
    assert len(w.layers) == len(ref.layers) == 3
    for (wa, ba), (wb, bb) in zip(w.layers, ref.layers):
        assert wa.tobytes() == np.asarray(wb, np.float32).tobytes()
        assert ba.tobytes() == np.asarray(bb, np.float32).tobytes()


@pytest.mark.parametrize("run", ["small_const", "velo_cos_wd"])
def test_checkpoint_load_save_cpu_bytes(tmp_path, run):
    """Reference checkpoint -> LearnedOptimizer (host tensors) -> checkpoint:
    the same bytes (params, accumulators, factors, step, schedule, decay)."""
    C = _C()
    src = os.path.join(GOLD, f"ref_ckpt_{run}.pylo")
    opt, params, names = C.checkpoint_load(src, device="cpu")
    assert opt.T == 3
    out = tmp_path / "ckpt.pylo"
    C.checkpoint_save(opt, out, names=names)
    assert out.read_bytes() == open(src, "rb").read()


def test_checkpoint_kind_checked(tmp_path):
    C = _C()
    with pytest.raises(C.CheckpointMismatchError):
        C.checkpoint_load(os.path.join(GOLD, "ref_weights_small_const.pylo"), device="cpu")
    with pytest.raises(C.CheckpointMismatchError):
        C.checkpoint_load(os.path.join(GOLD, "ref_ckpt_small_const.pylo"), device="cpu",
                          expect="velo_mlp")
