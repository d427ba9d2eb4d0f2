"""Sliced weight store and checkpoint loading.

The reference keeps weights as in-memory numpy arrays and re-slices them with
views on every ``slice_weights`` call (slicing_kernel.py:57-80); it has no
on-disk format and no checkpoint reader.  Here a placed layer is two byte
images -- the GG block as it sits in HBM and the pinned host region of CC and
CG chunks (see include/sliced.h) -- so the store is those images, 4 KB
aligned, behind one JSON header:

    b"SPSTORE1" | u64 header length | header JSON | pad to 4096 |
    for each layer: GG image | pad | host image | pad

Loading a layer is a ``pread`` straight into its pinned region plus one HBM
upload of the GG image (``sp_layer_load_file``): no repack, no extra copy.
Changing the rates later is ``NativeLayer.reslice`` (rows gathered back,
re-placed) -- measured by ``scripts/bench_store.py``.

Checkpoints: a dependency-free safetensors reader/writer (the format is an
8-byte little-endian header length, a JSON header of name -> dtype / shape /
byte offsets, then the raw tensor bytes) and a loader for HF Mixtral-layout MoE
layers (``model.layers.{l}.block_sparse_moe.{gate,experts.{e}.w1,w2,w3}``,
sharded through ``model.safetensors.index.json``).  bf16 tensors stay bf16 bit
patterns (uint16) from the file to the placed layer.
"""

from __future__ import annotations

import json
import os
import struct
from pathlib import Path
from typing import Iterable, Mapping, Sequence

import numpy as np

from .schedule import SlicingRates
from .sliced import NativeLayer, SlicedFFN, split_boundaries

MAGIC = b"SPSTORE1"
ALIGN = 4096


def _align(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


# ---------------------------------------------------------------------------
# sliced store


def save_store(path: str | os.PathLike, layers: Mapping[str, NativeLayer]) -> dict:
    """Write every layer's images behind one header; returns the header."""
    entries, images = {}, []
    for name, lay in layers.items():
        gg, host = lay.export_images()
        entries[name] = {"meta": lay.meta(), "gg_bytes": int(gg.size), "host_bytes": int(host.size)}
        images.append((name, gg, host))
    # offsets depend on the header length: size the header with placeholders first
    for e in entries.values():
        e["gg_offset"] = e["host_offset"] = 0
    header = {"format": "sliced-store", "version": 1, "layers": entries}
    hlen = len(json.dumps(header)) + 64 * (len(entries) + 1)  # room for the real offsets
    off = _align(len(MAGIC) + 8 + hlen)
    for name, gg, host in images:
        entries[name]["gg_offset"] = off
        off = _align(off + gg.size)
        entries[name]["host_offset"] = off
        off = _align(off + host.size)
    blob = json.dumps(header).encode()
    if len(blob) > hlen:
        raise RuntimeError("store header outgrew its reservation")
    blob = blob.ljust(hlen, b" ")
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<Q", hlen) + blob)
        for name, gg, host in images:
            e = entries[name]
            f.seek(e["gg_offset"])
            f.write(gg.tobytes())
            f.seek(e["host_offset"])
            f.write(host.tobytes())
        f.truncate(off)
    return header


def read_store_header(path: str | os.PathLike) -> dict:
    with open(path, "rb") as f:
        if f.read(len(MAGIC)) != MAGIC:
            raise ValueError(f"{path} is not a sliced store")
        (hlen,) = struct.unpack("<Q", f.read(8))
        return json.loads(f.read(hlen))


def load_store(path: str | os.PathLike, names: Iterable[str] | None = None,
               device: int | None = None) -> dict[str, NativeLayer]:
    """Recreate layers from a store (host image read straight into pinned memory)."""
    header = read_store_header(path)
    out = {}
    for name, e in header["layers"].items():
        if names is not None and name not in names:
            continue
        out[name] = NativeLayer.load_file(e["meta"], str(path), e["gg_offset"], e["gg_bytes"],
                                          e["host_offset"], e["host_bytes"], device=device)
    return out


# ---------------------------------------------------------------------------
# safetensors (no dependency on the safetensors package)

_ST_DTYPES = {"BF16": (np.uint16, 2), "F16": (np.float16, 2), "F32": (np.float32, 4), "F64": (np.float64, 8),
              "I32": (np.int32, 4), "I64": (np.int64, 8), "U8": (np.uint8, 1)}


def read_safetensors_header(path: str | os.PathLike) -> dict:
    with open(path, "rb") as f:
        (n,) = struct.unpack("<Q", f.read(8))
        return json.loads(f.read(n))


def load_safetensors(path: str | os.PathLike, names: Iterable[str] | None = None) -> dict[str, np.ndarray]:
    """name -> array (memory-mapped, read-only).  BF16 tensors come back as
    uint16 bit patterns, the form the runtime stores them in."""
    header = read_safetensors_header(path)
    with open(path, "rb") as f:
        (n,) = struct.unpack("<Q", f.read(8))
    base = 8 + n
    mm = np.memmap(path, dtype=np.uint8, mode="r")
    out = {}
    for name, info in header.items():
        if name == "__metadata__" or (names is not None and name not in names):
            continue
        dt, size = _ST_DTYPES[info["dtype"]]
        a, b = info["data_offsets"]
        if (b - a) != size * int(np.prod(info["shape"], dtype=np.int64)):
            raise ValueError(f"{path}:{name}: {b - a} bytes for shape {info['shape']} {info['dtype']}")
        out[name] = mm[base + a: base + b].view(dt).reshape(info["shape"])
    return out


def save_safetensors(path: str | os.PathLike, tensors: Mapping[str, np.ndarray],
                     dtypes: Mapping[str, str] | None = None) -> None:
    """Write tensors; ``dtypes[name] = "BF16"`` marks uint16 arrays as bf16 bits."""
    inv = {np.dtype(v[0]): k for k, v in _ST_DTYPES.items() if k != "BF16"}
    header, off, blobs = {}, 0, []
    for name, arr in tensors.items():
        arr = np.ascontiguousarray(arr)
        dt = (dtypes or {}).get(name) or inv[arr.dtype]
        header[name] = {"dtype": dt, "shape": list(arr.shape), "data_offsets": [off, off + arr.nbytes]}
        off += arr.nbytes
        blobs.append(arr)
    h = json.dumps(header).encode()
    h = h.ljust((len(h) + 7) // 8 * 8, b" ")
    with open(path, "wb") as f:
        f.write(struct.pack("<Q", len(h)) + h)
        for arr in blobs:
            f.write(arr.tobytes())


def _checkpoint_files(path: str | os.PathLike) -> dict[str, Path]:
    """tensor name -> file, for a single .safetensors file or an HF checkpoint dir."""
    p = Path(path)
    if p.is_file():
        return {name: p for name in read_safetensors_header(p) if name != "__metadata__"}
    index = p / "model.safetensors.index.json"
    if index.exists():
        return {k: p / v for k, v in json.loads(index.read_text())["weight_map"].items()}
    files = sorted(p.glob("*.safetensors"))
    return {name: f for f in files for name in read_safetensors_header(f) if name != "__metadata__"}


def load_tensors(path: str | os.PathLike, names: Sequence[str]) -> dict[str, np.ndarray]:
    where = _checkpoint_files(path)
    missing = [n for n in names if n not in where]
    if missing:
        raise KeyError(f"{path}: missing tensors {missing[:4]}{'...' if len(missing) > 4 else ''}")
    by_file: dict[Path, list[str]] = {}
    for n in names:
        by_file.setdefault(where[n], []).append(n)
    out = {}
    for f, ns in by_file.items():
        out.update(load_safetensors(f, ns))
    return out


def mixtral_moe_names(layer: int, n_experts: int, prefix: str = "model.layers") -> dict:
    base = f"{prefix}.{layer}.block_sparse_moe"
    return {"gate": f"{base}.gate.weight",
            "experts": [{w: f"{base}.experts.{e}.{w}.weight" for w in ("w1", "w2", "w3")} for e in range(n_experts)]}


def load_mixtral_moe(path: str | os.PathLike, layer: int, n_experts: int,
                     rates: SlicingRates | Sequence[SlicingRates], chunk_rows: int = 0,
                     device: int | None = None, prefix: str = "model.layers"):
    """Place one HF Mixtral-layout MoE layer: (experts, router [M, E] fp64).

    ``w1`` / ``w3`` are [H, M] (the runtime's W1t / W3t rows as stored), ``w2``
    is [M, H]; ``gate`` is [E, M].  ``rates`` may differ per expert."""
    names = mixtral_moe_names(layer, n_experts, prefix)
    wanted = [names["gate"]] + [n for e in names["experts"] for n in e.values()]
    t = load_tensors(path, wanted)
    per = list(rates) if isinstance(rates, (list, tuple)) else [rates] * n_experts
    dtype = "bf16" if t[names["experts"][0]["w1"]].dtype == np.uint16 else "f32"
    experts = []
    for e, nm in enumerate(names["experts"]):
        experts.append(SlicedFFN(t[nm["w1"]], t[nm["w2"]], per[e], w3t=t[nm["w3"]], activation="silu",
                                 dtype=dtype, chunk_rows=chunk_rows, device=device))
    gate = t[names["gate"]]
    if gate.dtype == np.uint16:
        gate = (gate.astype(np.uint32) << 16).view(np.float32)
    router = np.ascontiguousarray(np.asarray(gate, dtype=np.float64).T)
    return experts, router


__all__ = ["save_store", "load_store", "read_store_header", "load_safetensors", "save_safetensors",
           "read_safetensors_header", "load_tensors", "mixtral_moe_names", "load_mixtral_moe",
           "split_boundaries"]
