"""MOET trace codec (csrc/moet.cpp via the C ABI and paper_2602_00879_b200.moet)
vs the reference's own encoder / decoder (oracle/_ref: gen_trace,
encode_trace, decode_trace; trace.cpp:42-442).

CPU: encoded bytes are identical to the reference's for both formats; decoded
headers and logits are identical; every corruption (truncation at every
offset, byte flips, trailing data, JSONL edits) gives the reference's
TraceError code and message. GPU: decoded trace blocks route exactly like the
reference's routing of the same logits.
"""
import numpy as np
import pytest

from oracle.oracle import TraceDecodeError
from paper_2602_00879_b200 import moet

CASES = [  # (m, k, n, seed, rho, tau, model, layers, steps)
    (6, 2, 3, 8, 0.5, 1.0, "shared_bias", 1, 2),
    (14, 3, 5, 12345, 0.25, 1.5, "shared_bias", 2, 2),
    (64, 8, 32, 42, 0.3, 1.0, "shared_bias", 2, 3),
    (10, 2, 3, 99, 0.5, 2.0, "iid_gaussian", 1, 2),
    (10, 2, 3, 99, 0.5, 2.0, "dirichlet", 1, 2),
    (256, 8, 4, 7, 0.0, 0.7, "shared_bias", 1, 1),
]


def ours_or_error(data):
    try:
        f = moet.decode_trace(data)
        return ("ok", f)
    except moet.TraceError as e:
        return ("err", int(e.code), str(e))


def ref_or_error(ref, data):
    try:
        return ("ok", ref.trace_decode(data))
    except TraceDecodeError as e:
        return ("err", e.code, e.message)


def same_outcome(ref, data):
    a, b = ours_or_error(data), ref_or_error(ref, data)
    assert a[0] == b[0], (a, b)
    if a[0] == "err":
        assert a[1:] == b[1:], (a, b)
    else:
        f, (h, x) = a[1], b[1]
        assert (f.header.experts, f.header.top_k, f.header.layers, f.header.block_size,
                f.header.steps, int(f.header.model)) == (h["experts"], h["top_k"], h["layers"],
                                                         h["block_size"], h["steps"], h["model"])
        assert f.header.rho == h["rho"] and f.header.temperature == h["temperature"]
        assert f.header.seed == h["seed"]
        assert np.array_equal(np.stack([b.logits for b in f.blocks]), x)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("fmt", ["binary", "jsonl"])
def test_round_trip_bytes_identical_to_reference(ref, case, fmt):
    m, k, n, seed, rho, tau, model, layers, steps = case
    data = ref.trace_bytes(m, k, n, seed, rho=rho, tau=tau, model=model, layers=layers,
                           steps=steps, fmt=fmt)
    f = moet.decode_trace(data)
    assert f.block_count() == layers * steps
    assert moet.encode_trace(f, moet.TraceFormat[fmt]) == data
    same_outcome(ref, data)
    other = "jsonl" if fmt == "binary" else "binary"
    assert moet.encode_trace(f, moet.TraceFormat[other]) == ref.trace_bytes(
        m, k, n, seed, rho=rho, tau=tau, model=model, layers=layers, steps=steps, fmt=other)


def test_binary_truncation_every_offset(ref):
    data = ref.trace_bytes(6, 2, 3, 8, rho=0.5, steps=2)
    for cut in range(len(data)):
        same_outcome(ref, data[:cut])


def test_binary_corruptions(ref):
    data = bytearray(ref.trace_bytes(6, 2, 3, 8, rho=0.5, layers=2, steps=2))
    rng = np.random.default_rng(5)
    variants = [bytes(data) + b"zz", b"", b"M", b"XOET" + bytes(data[4:])]
    for pos, val in [(4, 9), (6, 3), (8, 0), (12, 9), (20, 0), (40, 1), (44, 7)]:
        v = bytearray(data)
        v[pos] = val
        variants.append(bytes(v))
    for _ in range(60):  # random byte flips in the records (keys, logits incl. NaN / Inf);
        # header sizes stay small: the reference allocates a record before reading it
        v = bytearray(data)
        v[int(rng.integers(40, len(v)))] = int(rng.integers(0, 256))
        variants.append(bytes(v))
    v = bytearray(data)
    v[-4:] = np.array([np.inf], np.float32).tobytes()
    variants.append(bytes(v))
    for d in variants:
        same_outcome(ref, d)


def test_jsonl_corruptions(ref):
    text = ref.trace_bytes(4, 2, 2, 3, rho=0.5, layers=1, steps=3, fmt="jsonl").decode()
    lines = text.split("\n")
    edits = [
        text.replace('"logits":[[', '"logits":[[0.0,', 1),             # 5-wide row
        "\n".join(lines[:-2]) + "\n",                                   # missing record 2
        text + "{}\n",                                                  # trailing data
        text + "\n\n",                                                  # trailing blank lines: fine
        text.replace('"version":1', '"version":2'),
        text.replace('"model":"shared_bias"', '"model":"bogus"'),
        text.replace('"experts":4', '"experts":0'),
        text.replace('"step":1', '"step":2', 1),
        text.replace('"logits":[[', '"logits":[["x",', 1),
        lines[0] + "\n" + "not json\n",
        "{not json\n",
        text.replace('"rho":0.5,', ''),
        text.replace('],[', '],[1.0],[', 1),
    ]
    for e in edits:
        same_outcome(ref, e.encode())


def test_header_encode_errors():
    f = moet.TraceFile(moet.TraceHeader(experts=4, top_k=5, layers=1, block_size=1, steps=1))
    with pytest.raises(moet.TraceError) as e:
        moet.encode_trace(f)
    assert e.value.code == moet.TraceError.Code.bad_header
    f = moet.TraceFile(moet.TraceHeader(experts=4, top_k=2, layers=1, block_size=1, steps=2))
    with pytest.raises(moet.TraceError) as e:
        moet.encode_trace(f)
    assert e.value.code == moet.TraceError.Code.shape_mismatch


def test_disk_round_trip(tmp_path, ref):
    data = ref.trace_bytes(6, 2, 2, 5, rho=0.75, steps=3)
    p = str(tmp_path / "t.moet")
    moet.write_trace(moet.decode_trace(data), p)
    assert open(p, "rb").read() == data
    assert moet.encode_trace(moet.read_trace(p)) == data
    with pytest.raises(moet.TraceError) as e:
        moet.read_trace(str(tmp_path / "missing.moet"))
    assert e.value.code == moet.TraceError.Code.io


@pytest.mark.gpu
def test_trace_blocks_route_like_reference(ref):
    from paper_2602_00879_b200 import dessim as ds
    data = ref.trace_bytes(64, 8, 32, 42, rho=0.3, layers=2, steps=2)
    f = moet.decode_trace(data)
    cfg = ds.PoolConfig(64, 8)
    for b in f.blocks:
        got = ds.des_run(b, cfg, ds.DesParams(ds.DesStrategy.vote, 1, 0.4))
        mem, r = ref.des_run(b.logits, 8, "vote", beta=0.4)
        assert got.coreset.members == mem.tolist()
        for t, tok in enumerate(got.assignment.tokens):
            assert tok.experts == r.experts(t)
            assert np.all(np.abs(np.array(tok.gates) - np.array(r.gates(t))) <= 1e-12)
