"""Circuit-set containers (reference container.py), B200 side: QGIR1 ingest.

The QGIR1 flat binary (container.py:1-16: magic, u32 capacity / n_circ /
n_meta, circ_type / gate_type / gate_param arrays, sorted meta pairs) is parsed
and written by libqgear_b200 (qg_qgir1_parse / qg_qgir1_write).  `read_arrays`
maps the file and returns zero-copy numpy views of the three arrays — they can
go straight to CompiledCircuit / qg_plan_create without one Python object per
gate (the reference's read_binary builds a GateRecord per padded slot).
`read_binary` / `write_binary` / `load_circuit_set` / `save_circuit_set` keep
the reference's names and behaviour (byte-identical files, ContainerFormatError
for bad magic / truncation / trailing bytes).  HDF5 needs h5py, which this
image does not have: those paths raise ContainerFormatError.
"""

from __future__ import annotations

import ctypes as C
import mmap
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import ContainerFormatError
from .ir import CircuitSet, set_from_arrays, set_to_arrays

FORMAT_VERSION = "1"
BINARY_MAGIC = b"QGIR1"
HDF5_MAGIC = b"\x89HDF"


def parse(buf) -> tuple[N.Qgir1Info, memoryview]:
    """Validate a QGIR1 image (bytes / mmap / buffer); return its layout."""
    mv = memoryview(buf).cast("B")
    raw = np.frombuffer(mv, dtype=np.uint8) if len(mv) else np.zeros(1, dtype=np.uint8)
    ptr = raw.ctypes.data_as(C.c_void_p)
    info = N.Qgir1Info()
    N.check(N.lib().qg_qgir1_parse(ptr, len(mv), C.byref(info)))
    return info, mv


def arrays_from_buffer(buf):
    """(circ_type (C,3) i32, gate_type (C,d,3) i32, gate_param (C,d) f64, metadata) as views of buf."""
    info, mv = parse(buf)
    raw = np.frombuffer(mv, dtype=np.uint8)
    nc, d = info.n_circ, info.capacity
    headers = np.frombuffer(raw, dtype="<i4", count=nc * 3, offset=info.headers_off).reshape(nc, 3)
    gate_type = np.frombuffer(raw, dtype="<i4", count=nc * d * 3, offset=info.gate_type_off).reshape(nc, d, 3)
    gate_param = np.frombuffer(raw, dtype="<f8", count=nc * d, offset=info.gate_param_off).reshape(nc, d)
    meta, off = {}, info.meta_off
    for _ in range(info.n_meta):
        kl = int.from_bytes(mv[off:off + 4], "little")
        key = bytes(mv[off + 4:off + 4 + kl]).decode("utf-8")
        off += 4 + kl
        vl = int.from_bytes(mv[off:off + 4], "little")
        meta[key] = bytes(mv[off + 4:off + 4 + vl]).decode("utf-8")
        off += 4 + vl
    return headers, gate_type, gate_param, meta


def read_arrays(path: str | Path):
    """Memory-map a QGIR1 file: zero-copy array views + metadata (see arrays_from_buffer)."""
    with open(path, "rb") as f:
        size = Path(path).stat().st_size
        if size == 0:
            raise ContainerFormatError("bad magic, not a QGIR1 file")
        mm = mmap.mmap(f.fileno(), 0, access=mmap.ACCESS_READ)
    return arrays_from_buffer(mm)


def encode_binary(circuit_set: CircuitSet) -> bytes:
    headers, gate_type, gate_param = set_to_arrays(circuit_set)
    items = sorted(circuit_set.metadata.items())
    raw = [t.encode("utf-8") for kv in items for t in kv]
    lens = np.array([len(r) for r in raw], dtype=np.int64)
    bufs = [C.create_string_buffer(r, len(r)) for r in raw]
    ptrs = (C.c_char_p * max(1, len(bufs)))(*[C.cast(b, C.c_char_p) for b in bufs])
    h = np.ascontiguousarray(headers, dtype="<i4")
    g = np.ascontiguousarray(gate_type, dtype="<i4")
    p = np.ascontiguousarray(gate_param, dtype="<f8")
    lib = N.lib()
    size = lib.qg_qgir1_size(circuit_set.capacity, h.shape[0], len(items), lens.ctypes.data_as(C.c_void_p))
    out = np.empty(size, dtype=np.uint8)
    N.check(lib.qg_qgir1_write(out.ctypes.data_as(C.c_void_p), size, circuit_set.capacity, h.shape[0],
                               h.ctypes.data_as(C.c_void_p), g.ctypes.data_as(C.c_void_p),
                               p.ctypes.data_as(C.c_void_p), len(items), C.cast(ptrs, C.c_void_p),
                               lens.ctypes.data_as(C.c_void_p)))
    return out.tobytes()


def write_binary(circuit_set: CircuitSet, path: str | Path) -> None:
    """container.py:71-84 (byte-identical output)."""
    Path(path).write_bytes(encode_binary(circuit_set))


def read_binary(path: str | Path) -> CircuitSet:
    """container.py:87-115."""
    headers, gate_type, gate_param, meta = read_arrays(path)
    return set_from_arrays(headers, gate_type, gate_param, meta)


def save_circuit_set(circuit_set: CircuitSet, path: str | Path) -> None:
    """container.py:118-123: HDF5 for .h5/.hdf5 (needs h5py), QGIR1 otherwise."""
    if Path(path).suffix.lower() in (".h5", ".hdf5"):
        raise ContainerFormatError("HDF5 containers need h5py, which is not installed; use a QGIR1 path")
    write_binary(circuit_set, path)


def load_circuit_set(path: str | Path) -> CircuitSet:
    """container.py:126-134: sniff the magic bytes."""
    with open(path, "rb") as f:
        head = f.read(8)
    if head.startswith(HDF5_MAGIC):
        raise ContainerFormatError(f"{path}: HDF5 container needs h5py, which is not installed")
    if head.startswith(BINARY_MAGIC):
        return read_binary(path)
    raise ContainerFormatError(f"{path}: unrecognized container format")
