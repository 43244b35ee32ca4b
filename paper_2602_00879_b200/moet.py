"""MOET router traces (the reference's trace.hpp / trace.cpp file format) on
the C ABI codec (csrc/moet.cpp: desmoe_moet_decode / desmoe_moet_encode).

Mirror of the reference API: TraceHeader, TraceFile, TraceFormat,
TraceError (with .code = TraceError::Code), encode_trace, decode_trace,
write_trace, read_trace. Decoded blocks are dessim.RouterBlock values that
feed the GPU routing entry points directly (logits in); see
tools/route_trace.py. The codec is host code: no GPU needed.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _lib
from .dessim import RouterBlock


class SynthModel(enum.IntEnum):  # trace.hpp:13
    iid_gaussian = 0
    dirichlet = 1
    shared_bias = 2


class TraceFormat(enum.IntEnum):  # trace.hpp:55
    binary = _lib.MOET_BINARY
    jsonl = _lib.MOET_JSONL


class TraceError(RuntimeError):
    """trace.hpp:58-71; .code is the TraceError::Code ordinal."""

    class Code(enum.IntEnum):
        io = 0
        bad_magic = 1
        bad_version = 2
        bad_header = 3
        truncated = 4
        shape_mismatch = 5
        bad_value = 6

    def __init__(self, code, message):
        super().__init__(message)
        self.code = TraceError.Code(code)


@dataclass
class TraceHeader:  # trace.hpp:29-39
    experts: int = 0
    top_k: int = 0
    layers: int = 0
    block_size: int = 0
    steps: int = 0
    model: SynthModel = SynthModel.iid_gaussian
    rho: float = 0.0
    temperature: float = 1.0
    seed: int = 0


@dataclass
class TraceFile:  # trace.hpp:41-49, blocks in (step, layer) order
    header: TraceHeader
    blocks: List[RouterBlock] = field(default_factory=list)

    def block(self, step: int, layer: int) -> RouterBlock:
        h = self.header
        if step < 0 or step >= h.steps or layer < 0 or layer >= h.layers:
            raise ValueError("block key out of range")
        return self.blocks[step * h.layers + layer]

    def block_count(self) -> int:
        return len(self.blocks)


def _c_header(h: TraceHeader) -> _lib.MoetHeader:
    return _lib.MoetHeader(h.experts, h.top_k, h.layers, h.block_size, h.steps, int(h.model),
                           h.rho, h.temperature, h.seed)


def _raise(code: C.c_int):
    raise TraceError(max(code.value, 0), _lib.lib().desmoe_last_error().decode())


def decode_trace(data: bytes) -> TraceFile:
    """trace.cpp:432-441 (binary or JSONL, sniffed)."""
    L = _lib.lib()
    h = _lib.MoetHeader()
    code = C.c_int()
    buf = C.create_string_buffer(bytes(data), len(data))
    if L.desmoe_moet_decode(buf, len(data), C.byref(h), None, C.byref(code)):
        _raise(code)
    x = np.empty((h.steps * h.layers, h.block_size, h.experts), np.float64)
    if L.desmoe_moet_decode(buf, len(data), C.byref(h), x.ctypes.data, C.byref(code)):
        _raise(code)
    head = TraceHeader(h.experts, h.top_k, h.layers, h.block_size, h.steps, SynthModel(h.model),
                       h.rho, h.temperature, h.seed)
    return TraceFile(head, [RouterBlock(h.block_size, h.experts, x[r].copy())
                            for r in range(x.shape[0])])


def encode_trace(f: TraceFile, fmt: TraceFormat = TraceFormat.binary) -> bytes:
    """trace.cpp:422-430."""
    L = _lib.lib()
    h = _c_header(f.header)
    code = C.c_int()
    n = C.c_size_t(0)
    if L.desmoe_moet_encode(C.byref(h), None, int(fmt), None, C.byref(n), C.byref(code)):
        _raise(code)
    if f.block_count() != f.header.steps * f.header.layers:
        raise TraceError(TraceError.Code.shape_mismatch, "block count does not match header")
    x = np.ascontiguousarray(np.stack([np.asarray(b.logits, np.float64).reshape(-1)
                                       for b in f.blocks]), np.float64)
    if L.desmoe_moet_encode(C.byref(h), x.ctypes.data, int(fmt), None, C.byref(n), C.byref(code)):
        _raise(code)
    out = C.create_string_buffer(n.value)
    if L.desmoe_moet_encode(C.byref(h), x.ctypes.data, int(fmt), out, C.byref(n), C.byref(code)):
        _raise(code)
    return out.raw[: n.value]


def write_trace(f: TraceFile, path: str, fmt: TraceFormat = TraceFormat.binary):
    data = encode_trace(f, fmt)
    try:
        with open(path, "wb") as fh:
            fh.write(data)
    except OSError as e:
        raise TraceError(TraceError.Code.io, f"cannot open for writing: {path}") from e


def read_trace(path: str) -> TraceFile:
    try:
        with open(path, "rb") as fh:
            data = fh.read()
    except OSError as e:
        raise TraceError(TraceError.Code.io, f"cannot open for reading: {path}") from e
    return decode_trace(data)
