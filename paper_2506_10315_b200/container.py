"""The reference's named-tensor container ("PYLO" v1) and its checkpoint /
weights layout, so GPU optimizers read and write the reference's files.

File layout (pkg/src/lopt/tensors.py:1-20): magic b"PYLO", u32 LE version 1,
u64 LE header length, a UTF-8 JSON header {"entries": [{name, dtype, shape,
offset, nbytes}], "meta": {str: str}}, then the little-endian payload with
every buffer at an 8-byte aligned offset relative to the payload start.
dtype tags: f32, f64, i64.

Layouts on top of it:
  * weights (engine.py:195-250): entries mlp/w{i}, mlp/b{i}; meta n_layers,
    alpha, beta_out, update_sign, momentum_betas, second_moment_beta,
    adafactor_betas, kind="lopt_weights", feature_set;
  * checkpoint (optim.py:224-282): param/<name>, state/<name>/{M0,M1,M2,V,
    r0,r1,r2,c0,c1,c2,t} (state.py:133-154) plus the weights, meta kind=
    "checkpoint", step, feature_set, tensors (JSON list of names), schedule
    fields, weight_decay, path, workers.

The writer emits the same bytes as the reference for the same entries and
meta (same JSON serialization, same padding), so files compare bitwise.
"""

from __future__ import annotations

import io
import json
import struct

import numpy as np

MAGIC = b"PYLO"
VERSION = 1
_TAGS = {"f32": np.dtype("<f4"), "f64": np.dtype("<f8"), "i64": np.dtype("<i8")}
_MAX_ELEMENTS = 1 << 40


class FileFormatError(Exception):
    """tensors.py:50 -- base class of container problems."""


class VersionMismatchError(FileFormatError):
    """Unsupported format version."""


class TruncatedFileError(FileFormatError):
    """The file ends before its header or a payload does."""


class MalformedHeaderError(FileFormatError):
    """Bad magic, bad JSON, or inconsistent entry records."""


class CheckpointMismatchError(Exception):
    """optim.py: the file is not a checkpoint, or for another feature set."""


def _tag(a: np.ndarray) -> str:
    kind, size = a.dtype.kind, a.dtype.itemsize
    if kind == "f" and size == 4:
        return "f32"
    if kind == "f" and size == 8:
        return "f64"
    if kind == "i" and size == 8:
        return "i64"
    raise ValueError(f"dtype {a.dtype} is not storable in a PYLO container (f32, f64, i64)")


def file_save(entries: dict, meta: dict, path) -> None:
    """Named arrays + string metadata -> PYLO v1 file."""
    records, blobs, off = [], [], 0
    for name, arr in entries.items():
        if not isinstance(name, str) or not name:
            raise ValueError(f"bad entry name {name!r}")
        a = np.asarray(arr)
        shape = list(a.shape)
        tag = _tag(a)
        raw = np.ascontiguousarray(a).astype(_TAGS[tag], copy=False).tobytes()
        off = (off + 7) // 8 * 8
        records.append({"name": name, "dtype": tag, "shape": shape, "offset": off,
                        "nbytes": len(raw)})
        blobs.append((off, raw))
        off += len(raw)
    header = json.dumps({"entries": records, "meta": {str(k): str(v) for k, v in meta.items()}},
                        ensure_ascii=False).encode("utf-8")
    payload = bytearray(off)
    for o, raw in blobs:
        payload[o:o + len(raw)] = raw
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<IQ", VERSION, len(header)) + header + bytes(payload))


def file_load(path):
    """PYLO v1 file -> (entries, meta); typed errors as tensors.py:169-230."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 16:
        raise TruncatedFileError(f"{path}: shorter than the 16-byte preamble")
    if data[:4] != MAGIC:
        raise MalformedHeaderError(f"{path}: magic {data[:4]!r} is not {MAGIC!r}")
    version, hlen = struct.unpack_from("<IQ", data, 4)
    if version != VERSION:
        raise VersionMismatchError(f"{path}: format version {version}, supported {VERSION}")
    if len(data) < 16 + hlen:
        raise TruncatedFileError(f"{path}: header runs past the end of the file")
    try:
        header = json.loads(data[16:16 + hlen].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as e:
        raise MalformedHeaderError(f"{path}: header is not JSON ({e})") from e
    if not isinstance(header, dict) or "entries" not in header or "meta" not in header:
        raise MalformedHeaderError(f"{path}: header lacks entries/meta")
    payload = memoryview(data)[16 + hlen:]
    entries = {}
    for rec in header["entries"]:
        try:
            name, tag = rec["name"], rec["dtype"]
            shape = tuple(int(x) for x in rec["shape"])
            off, nbytes = int(rec["offset"]), int(rec["nbytes"])
        except (KeyError, TypeError, ValueError) as e:
            raise MalformedHeaderError(f"{path}: bad entry record {rec!r}") from e
        if tag not in _TAGS:
            raise MalformedHeaderError(f"{path}: unknown dtype tag {tag!r}")
        if name in entries:
            raise MalformedHeaderError(f"{path}: duplicate entry {name!r}")
        count = int(np.prod(shape, dtype=np.int64)) if shape else 1
        if count > _MAX_ELEMENTS or count * _TAGS[tag].itemsize != nbytes:
            raise MalformedHeaderError(f"{path}: entry {name!r}: shape {shape} vs {nbytes} bytes")
        if off % 8:
            raise MalformedHeaderError(f"{path}: entry {name!r} offset {off} not 8-byte aligned")
        if off + nbytes > len(payload):
            raise TruncatedFileError(f"{path}: entry {name!r} runs past the end of the file")
        entries[name] = np.frombuffer(payload, _TAGS[tag], count, off).reshape(shape).copy()
    return entries, {str(k): str(v) for k, v in header["meta"].items()}


# ---------------------------------------------------------------------------
# weights (engine.py:195-250)

def weights_entries(w):
    entries = {}
    for i, (wt, b) in enumerate(w.layers):
        entries[f"mlp/w{i}"] = wt
        entries[f"mlp/b{i}"] = b
    meta = {
        "n_layers": str(w.n_layers),
        "alpha": repr(float(w.alpha)),
        "beta_out": repr(float(w.beta_out)),
        "update_sign": str(w.update_sign),
        "momentum_betas": ",".join(repr(float(b)) for b in w.betas.momentum_betas),
        "second_moment_beta": repr(float(w.betas.second_moment_beta)),
        "adafactor_betas": ",".join(repr(float(b)) for b in w.betas.adafactor_betas),
    }
    return entries, meta


def weights_from_entries(entries, meta):
    from .weights import BetaConfig, LoptWeights

    n = int(meta["n_layers"])
    betas = BetaConfig(
        momentum_betas=tuple(float(x) for x in meta["momentum_betas"].split(",")),
        second_moment_beta=float(meta["second_moment_beta"]),
        adafactor_betas=tuple(float(x) for x in meta["adafactor_betas"].split(",")))
    return LoptWeights(layers=[(entries[f"mlp/w{i}"], entries[f"mlp/b{i}"]) for i in range(n)],
                       alpha=float(meta["alpha"]), beta_out=float(meta["beta_out"]), betas=betas,
                       update_sign=int(meta["update_sign"]))


def save_weights(w, feature_set: str, path) -> None:
    entries, meta = weights_entries(w)
    meta["kind"] = "lopt_weights"
    meta["feature_set"] = feature_set
    file_save(entries, meta, path)


def load_weights(path, expect: str | None = None):
    """-> (LoptWeights, feature_set name)."""
    from .features import spec_by_name

    entries, meta = file_load(path)
    fs = meta.get("feature_set")
    if fs is None:
        raise MalformedHeaderError(f"{path}: no feature_set in the metadata")
    if expect is not None and fs != expect:
        raise MalformedHeaderError(f"weights are for feature set {fs!r}, expected {expect!r}")
    w = weights_from_entries(entries, meta)
    if w.input_dim != spec_by_name(fs).d_feat:
        raise MalformedHeaderError(f"MLP input dim {w.input_dim} does not match {fs!r}")
    return w, fs


# ---------------------------------------------------------------------------
# checkpoints (optim.py:224-282, state.py:133-154)

def state_entries(prefix, quad, r, c, m, n, t):
    """Our packed {M1,M2,M3,V} quads + factors -> the reference's entries."""
    q = np.asarray(quad, np.float32).reshape(m * n, 4)
    out = {}
    for i in range(3):
        out[f"{prefix}/M{i}"] = q[:, i].reshape(m, n)
    out[f"{prefix}/V"] = q[:, 3].reshape(m, n)
    for i in range(3):
        out[f"{prefix}/r{i}"] = np.asarray(r, np.float32)[i]
        out[f"{prefix}/c{i}"] = np.asarray(c, np.float32)[i]
    out[f"{prefix}/t"] = np.array([[t]], dtype=np.int64)
    return out


def state_from_entries(prefix, entries, m, n):
    """-> (quad (m*n, 4), r (3, m), c (3, n), t)."""
    quad = np.empty((m * n, 4), np.float32)
    for i in range(3):
        quad[:, i] = entries[f"{prefix}/M{i}"].astype(np.float32).reshape(-1)
    quad[:, 3] = entries[f"{prefix}/V"].astype(np.float32).reshape(-1)
    r = np.stack([entries[f"{prefix}/r{i}"].astype(np.float32).ravel() for i in range(3)])
    c = np.stack([entries[f"{prefix}/c{i}"].astype(np.float32).ravel() for i in range(3)])
    t = int(entries[f"{prefix}/t"].ravel()[0])
    return quad, r, c, t


def checkpoint_save(opt, path, names=None) -> None:
    """A LearnedOptimizer (one parameter group) -> reference checkpoint file.
    `names`: tensor names (default t0, t1, ...)."""
    from .optim import view_2d

    ps = [p for g in opt.param_groups for p in g["params"]]
    names = list(names) if names is not None else [f"t{k}" for k in range(len(ps))]
    if len(names) != len(ps):
        raise ValueError(f"{len(names)} names for {len(ps)} tensors")
    if getattr(opt, "hypernet", None) is not None:
        raise ValueError("the PYLO checkpoint layout has no VeLO hypernetwork state "
                         "(optim.py:224-282); use opt.state_dict()")
    for p in ps:
        rng_ = opt.state.get(p, {}).get("range")
        if rng_ is not None and tuple(rng_) != (0, p.numel()):
            raise ValueError("sharded optimizer state covers only this rank's element range; "
                             "save per rank with state_dict() or gather it first")
    entries = {}
    for name, p in zip(names, ps):
        entries[f"param/{name}"] = p.detach().cpu().numpy().reshape(view_2d(p.shape))
    for name, p in zip(names, ps):
        m, n = view_2d(p.shape)
        st = opt.state.get(p, {})
        if "quad" in st:
            quad = st["quad"].cpu().numpy()
            r, c = st["row_factors"].cpu().numpy(), st["col_factors"].cpu().numpy()
        else:
            quad = np.zeros((m * n, 4), np.float32)
            r, c = np.zeros((3, m), np.float32), np.zeros((3, n), np.float32)
        entries.update(state_entries(f"state/{name}", quad, r, c, m, n, opt.T))
    w_entries, w_meta = weights_entries(opt.lopt_weights)
    entries.update(w_entries)
    meta = dict(w_meta)
    group = opt.param_groups[0]
    sch = opt.schedule
    meta.update({
        "kind": "checkpoint",
        "step": str(opt.T),
        "feature_set": opt.spec.id.value,
        "tensors": json.dumps(names),
        "schedule_kind": sch.kind if sch is not None else "constant",
        "max_lr": repr(float(sch.max_lr if sch is not None else group["lr"])),
        "min_lr": repr(float(sch.min_lr if sch is not None else 0.0)),
        "warmup_steps": str(sch.warmup_steps if sch is not None else 0),
        "total_steps": str(sch.total_steps if sch is not None else 1),
        "weight_decay": repr(float(group["weight_decay"])),
        "path": "fused",
        "workers": "1",
    })
    file_save(entries, meta, path)


def checkpoint_load(path, device="cuda", mode="strict", expect: str | None = None, **kw):
    """Reference checkpoint -> (LearnedOptimizer, params, names): parameters
    as CUDA tensors of the stored 2-D shapes, accumulators, factors, step
    counter, schedule and weight decay restored, so the next step continues
    the reference's trajectory (bitwise in strict mode)."""
    import torch

    from .features import spec_by_name
    from .optim import LearnedOptimizer
    from .schedule import ScheduleConfig

    entries, meta = file_load(path)
    if meta.get("kind") != "checkpoint":
        raise CheckpointMismatchError(f"not a checkpoint file: kind={meta.get('kind')!r}")
    fs = meta["feature_set"]
    if expect is not None and fs != expect:
        raise CheckpointMismatchError(f"checkpoint feature set {fs!r}, expected {expect!r}")
    spec = spec_by_name(fs)
    w = weights_from_entries(entries, meta)
    names = json.loads(meta["tensors"])
    T = int(meta["step"])
    sched = ScheduleConfig(kind=meta["schedule_kind"], max_lr=float(meta["max_lr"]),
                           min_lr=float(meta["min_lr"]), warmup_steps=int(meta["warmup_steps"]),
                           total_steps=int(meta["total_steps"]))
    params = [torch.nn.Parameter(torch.from_numpy(
        np.ascontiguousarray(entries[f"param/{nm}"], np.float32)).to(device)) for nm in names]
    schedule = None if sched.kind == "constant" else sched
    opt = LearnedOptimizer(params, lr=sched.max_lr, weight_decay=float(meta["weight_decay"]),
                           feature_set=spec.id.value, weights=w, schedule=schedule, mode=mode, **kw)
    for nm, p in zip(names, params):
        m, n = p.shape
        quad, r, c, t = state_from_entries(f"state/{nm}", entries, m, n)
        if t != T:
            raise CheckpointMismatchError(f"tensor {nm!r}: state t={t} but step {T}")
        st = opt.state[p]
        st["quad"] = torch.from_numpy(quad).to(device)
        st["row_factors"] = torch.from_numpy(r).to(device)
        st["col_factors"] = torch.from_numpy(c).to(device)
        st["step"] = T
    opt.T = T
    return opt, params, names


def dumps(entries, meta) -> bytes:
    """Serialized file image (tests compare writers byte for byte)."""
    buf = io.BytesIO()
    import os
    import tempfile

    with tempfile.NamedTemporaryFile(delete=False) as f:
        tmp = f.name
    try:
        file_save(entries, meta, tmp)
        with open(tmp, "rb") as f:
            buf.write(f.read())
    finally:
        os.unlink(tmp)
    return buf.getvalue()
