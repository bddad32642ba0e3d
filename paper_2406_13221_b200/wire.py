"""Ciphertext / key wire format.

The reference stores a packed (plaintext) matrix as a JSON manifest plus an
``npz`` of slot vectors (``save_packed`` / ``load_packed``,
encoding.py:160-206); ``save_packed`` / ``load_packed`` below keep that exact
layout, so the files are interchangeable.  Encrypted data has no reference
counterpart (the simulator never leaves Python), so the real-CKKS objects get
a limb-major binary format with a manifest:

* ``manifest.json`` — format tag and version, the ring (log N, the q and p
  primes, dnum), and one record per ciphertext group: name, shape, level,
  scale, byte offset and length in ``data.bin``;
* ``data.bin`` — little-endian u64 residues.  A ciphertext group of shape
  (..., 2, L, N) at level l stores only limbs 0..l of every polynomial,
  polynomial-major then limb-major, so a level-l ciphertext costs
  2 (l+1) N 8 bytes;
* evaluation keys are groups of shape (beta, 2, L+K, N), stored whole, tagged
  with their Galois element (0 = relinearisation key).

Loading checks the ring against the receiving context (a key or ciphertext
is meaningless under other primes) and copies through pinned host memory.
The format is host I/O; the device never sees it.
"""

from __future__ import annotations

import json
from pathlib import Path
from typing import Dict, Iterable, Optional

import numpy as np
import torch

__all__ = ["save_packed", "load_packed", "CipherStore", "save_keys", "load_keys",
           "save_trainer_data", "load_trainer_data", "FORMAT", "VERSION"]

FORMAT = "helr-b200-rns-ckks"
VERSION = 1


# ------------------------------------------------------------ plaintext (reference layout)
def save_packed(directory, blocks, layout) -> None:
    """Manifest (JSON) plus binary slot dumps for a packed matrix; the same
    files as the reference's ``save_packed`` (encoding.py:160-184)."""
    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    manifest = {
        "n": layout.n, "f": layout.f, "m": layout.m, "g": layout.g,
        "row_blocks": layout.row_blocks, "col_blocks": layout.col_blocks,
        "blocks": [{"row": i, "col": j, "key": f"block_{i}_{j}"}
                   for i in range(layout.row_blocks) for j in range(layout.col_blocks)],
    }
    with open(directory / "manifest.json", "w", encoding="utf-8") as fh:
        json.dump(manifest, fh, indent=2)
    arrays = {f"block_{i}_{j}": np.asarray(blocks[i][j])
              for i in range(layout.row_blocks) for j in range(layout.col_blocks)}
    np.savez(directory / "blocks.npz", **arrays)


def load_packed(directory):
    """Inverse of ``save_packed`` (encoding.py:187-206)."""
    from .encoding import BlockLayout
    directory = Path(directory)
    with open(directory / "manifest.json", "r", encoding="utf-8") as fh:
        mf = json.load(fh)
    layout = BlockLayout(n=mf["n"], f=mf["f"], m=mf["m"], g=mf["g"], row_blocks=mf["row_blocks"],
                         col_blocks=mf["col_blocks"], pad_rows=mf["row_blocks"] * mf["m"] - mf["n"],
                         pad_cols=mf["col_blocks"] * mf["g"] - (mf["f"] + 1))
    with np.load(directory / "blocks.npz") as arrays:
        blocks = [[arrays[f"block_{i}_{j}"] for j in range(layout.col_blocks)] for i in range(layout.row_blocks)]
    return blocks, layout


# ------------------------------------------------------------ encrypted objects
def _ring(ck) -> dict:
    return {"log_n": int(ck.log_n), "q": [int(x) for x in ck.q], "p": [int(x) for x in ck.p], "dnum": int(ck.dnum)}


class CipherStore:
    """A directory of ciphertext groups and keys (manifest.json + data.bin).

    Write: ``CipherStore.create(dir, ckks)``, then ``put(...)``, then
    ``close()``.  Read: ``CipherStore.open(dir)``, then ``get(name, device)``.
    """

    def __init__(self, directory, manifest: dict, mode: str):
        self.dir = Path(directory)
        self.manifest = manifest
        self.mode = mode
        self._fh = open(self.dir / "data.bin", "wb" if mode == "w" else "rb")

    @classmethod
    def create(cls, directory, ckks) -> "CipherStore":
        d = Path(directory)
        d.mkdir(parents=True, exist_ok=True)
        return cls(d, {"format": FORMAT, "version": VERSION, "ring": _ring(ckks), "groups": []}, "w")

    @classmethod
    def open(cls, directory) -> "CipherStore":
        d = Path(directory)
        with open(d / "manifest.json", "r", encoding="utf-8") as fh:
            mf = json.load(fh)
        if mf.get("format") != FORMAT:
            raise ValueError(f"{d}: not a {FORMAT} store")
        if mf.get("version") != VERSION:
            raise ValueError(f"{d}: unsupported version {mf.get('version')}")
        return cls(d, mf, "r")

    def check_ring(self, ckks) -> None:
        if self.manifest["ring"] != _ring(ckks):
            raise ValueError("stored ring (primes / N / dnum) differs from the context's")

    @property
    def names(self) -> list:
        return [g["name"] for g in self.manifest["groups"]]

    def put(self, name: str, t: torch.Tensor, level: Optional[int] = None, scale: Optional[float] = None,
            kind: str = "ct", meta: Optional[dict] = None) -> None:
        """Append a group.  kind "ct": shape (..., 2, L, N), limbs 0..level
        stored; kind "key": stored whole."""
        if self.mode != "w":
            raise ValueError("store opened read-only")
        if name in self.names:
            raise ValueError(f"duplicate group {name!r}")
        a = t.detach().to("cpu").contiguous().numpy().view(np.uint64)
        shape = list(a.shape)
        if kind == "ct":
            if a.ndim < 3 or shape[-3] != 2:
                raise ValueError("ciphertext groups have shape (..., 2, L, N)")
            L = shape[-2]
            lv = L - 1 if level is None else int(level)
            if not 0 <= lv < L:
                raise ValueError(f"level {lv} outside [0, {L})")
            a = a[..., : lv + 1, :]
        else:
            lv = None
        off = self._fh.tell()
        data = np.ascontiguousarray(a).astype("<u8", copy=False)
        data.tofile(self._fh)
        self.manifest["groups"].append({"name": name, "kind": kind, "shape": shape, "level": lv,
                                        "scale": None if scale is None else float(scale), "offset": off,
                                        "nbytes": int(data.nbytes), "meta": meta or {}})

    def info(self, name: str) -> dict:
        for g in self.manifest["groups"]:
            if g["name"] == name:
                return g
        raise KeyError(name)

    def get(self, name: str, device="cpu", out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """The group as an int64 tensor of its full shape (inactive limbs of a
        ciphertext group are zero), on ``device`` (or copied into ``out``)."""
        g = self.info(name)
        shape = g["shape"]
        stored = list(shape)
        if g["kind"] == "ct":
            stored[-2] = g["level"] + 1
        cnt = int(np.prod(stored))
        if cnt * 8 != g["nbytes"]:
            raise ValueError(f"{name}: manifest size mismatch")
        self._fh.seek(g["offset"])
        raw = np.fromfile(self._fh, dtype="<u8", count=cnt)
        if raw.size != cnt:
            raise ValueError(f"{name}: data.bin truncated")
        host = torch.zeros(shape, dtype=torch.int64, pin_memory=torch.cuda.is_available())
        src = torch.from_numpy(raw.view(np.int64).reshape(stored))
        if g["kind"] == "ct":
            host[..., : g["level"] + 1, :].copy_(src)
        else:
            host.copy_(src)
        if out is not None:
            if list(out.shape) != shape:
                raise ValueError(f"{name}: destination shape {list(out.shape)} != {shape}")
            out.copy_(host)
            return out
        return host.to(device)

    def close(self) -> None:
        if self._fh is not None:
            self._fh.close()
            self._fh = None
        if self.mode == "w":
            with open(self.dir / "manifest.json", "w", encoding="utf-8") as fh:
                json.dump(self.manifest, fh, indent=1)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ------------------------------------------------------------ keys
def save_keys(directory, ctx, galois: Optional[Iterable[int]] = None) -> None:
    """Relinearisation key + Galois keys of a GpuContext (the evaluation key
    set a client ships to the server; the secret key is never written)."""
    gal = sorted(ctx._gks) if galois is None else [int(g) % (2 * ctx.ckks.n) for g in galois]
    with CipherStore.create(directory, ctx.ckks) as st:
        st.put("rlk", ctx.rlk, kind="key", meta={"galois": 0})
        for g in gal:
            st.put(f"gk_{g}", ctx.galois_key(g), kind="key", meta={"galois": g})


def load_keys(directory, ctx) -> Dict[int, torch.Tensor]:
    """Install stored evaluation keys into ``ctx`` (replacing its own)."""
    with CipherStore.open(directory) as st:
        st.check_ring(ctx.ckks)
        ctx.rlk = st.get("rlk", ctx.device)
        out = {}
        for g in st.manifest["groups"]:
            if g["kind"] == "key" and g["meta"].get("galois", 0) != 0:
                out[int(g["meta"]["galois"])] = st.get(g["name"], ctx.device)
        ctx._gks.update(out)
    return out


# ------------------------------------------------------------ a trainer's encrypted dataset
def save_trainer_data(directory, tr) -> None:
    """The encrypted dataset (Z blocks), B̄ ciphertexts and W, V of a
    FusedTrainer, with their scales, the block layout and the iteration's
    schedule state (t, alpha), so training resumes where it stopped."""
    lay = tr.layout
    meta = {"layout": {k: int(getattr(lay, k)) for k in ("n", "f", "m", "g", "row_blocks", "col_blocks",
                                                         "pad_rows", "pad_cols")},
            "mode": tr.mode, "rows": tr.rows, "n_batches": tr.n_batches,
            # host-side schedule state of the NAG iteration
            "t": int(tr.t), "alpha0": float(tr.alpha0), "alpha1": float(tr.alpha1),
            # encryption-nonce counter of the context (refresh re-encryptions):
            # a resumed run continues it and never reuses a nonce
            "ct_id": int(tr.ctx._next_ct_id)}
    with CipherStore.create(directory, tr.ck) as st:
        st.put("z", tr.z, level=tr.ck.top_level, scale=tr.s_z, meta=meta)
        st.put("bbar", tr.bbar, level=tr.ck.top_level, scale=tr.s_b)
        st.put("wv", tr.wv, level=tr.level, scale=tr.s_w)


def load_trainer_data(directory, tr) -> None:
    """Replace a FusedTrainer's encrypted dataset / B̄ / W, V with stored
    ones (same ring and layout required)."""
    with CipherStore.open(directory) as st:
        st.check_ring(tr.ck)
        zi = st.info("z")
        lay = zi["meta"]["layout"]
        mine = {k: int(getattr(tr.layout, k)) for k in lay}
        if lay != mine or zi["shape"] != list(tr.z.shape):
            raise ValueError("stored dataset layout differs from the trainer's")
        st.get("z", out=tr.z)
        st.get("bbar", out=tr.bbar)
        st.get("wv", out=tr.wv)
        tr.s_z, tr.s_b = zi["scale"], st.info("bbar")["scale"]
        m = zi["meta"]
        tr.t, tr.alpha0, tr.alpha1 = m["t"], m["alpha0"], m["alpha1"]
        tr.ctx._next_ct_id = max(tr.ctx._next_ct_id, int(m["ct_id"]))
        wi = st.info("wv")
        tr.level, tr.s_w = wi["level"], wi["scale"]
        tr.s_v = tr.s_w
