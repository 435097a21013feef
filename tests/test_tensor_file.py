"""APMM v1 tensor files (reference tensor_file.hpp:12-64,
tensor_file.cpp:124-229): the C library's parser against the reference's own golden bytes
(test_tensor_file.cpp:21-26) and against files the reference's serializer wrote
(tests/golden/*.apmm, oracle/gen_golden.py), error classes against the reference library on
the same corrupt bytes, and -- on the GPU -- the device upload equal to to_packed()."""
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")

# test_tensor_file.cpp:21-26: header, one f64 scale of 1.0, plane words 0b0011, 0b0101
GOLDEN_BYTES = bytes([0x41, 0x50, 0x4D, 0x4D, 0x01, 0x01, 0x02, 0x00,
                      0x01, 0x00, 0x00, 0x00, 0x04, 0x00, 0x00, 0x00,
                      0x00, 0x00, 0x00, 0x00, 0x00, 0x00, 0xF0, 0x3F,
                      0x03, 0x00, 0x00, 0x00, 0x05, 0x00, 0x00, 0x00])


@pytest.fixture(scope="module")
def ap():
    import paper_2409_17870_b200 as ap
    return ap


def test_golden_bytes_parse(ap):
    # test_tensor_file.cpp:38-48
    t = ap.parse_tensor(GOLDEN_BYTES)
    assert t.kind == ap.TensorKind.QuantizedBipolar and t.bit_width == 2
    assert t.granularity_enum() == ap.Granularity.PerTensor
    assert (t.rows, t.cols) == (1, 4)
    assert t.scales.tolist() == [1.0] and t.packed.tolist() == [0b0011, 0b0101]
    assert ap.serialize_tensor(t) == GOLDEN_BYTES
    assert open(os.path.join(GOLD, "w2_1x4_tensor.apmm"), "rb").read() == GOLDEN_BYTES


def test_reference_written_files_parse_exactly(ap, golden):
    for f in golden["tensor_files"]:
        data = open(os.path.join(GOLD, f["file"]), "rb").read()
        t = ap.parse_tensor(data)
        assert (t.rows, t.cols, int(t.kind)) == (f["rows"], f["cols"], f["kind"])
        if f["kind"] == 1:
            assert t.bit_width == f["n"] and t.granularity == f["gran"]
            assert t.packed.tolist() == f["words"]
            assert [float(v).hex() for v in t.scales] == f["scales"]
            assert ap.serialize_tensor(t) == data  # byte-identical re-serialization
            assert t.to_packed().words().tolist() == f["words"]
        else:
            assert [float(v).hex() for v in t.to_real().reshape(-1)] == f["values"]


def _corrupt_cases():
    g = bytearray(GOLDEN_BYTES)
    cases = {"truncated header": bytes(g[:10]), "bad magic": b"APMX" + bytes(g[4:])}
    b = bytearray(g); b[4] = 2; cases["version"] = bytes(b)
    b = bytearray(g); b[5] = 7; cases["kind"] = bytes(b)
    b = bytearray(g); b[6] = 9; cases["width"] = bytes(b)
    b = bytearray(g); b[7] = 3; cases["granularity"] = bytes(b)
    b = bytearray(g); b[8] = 0; cases["zero rows"] = bytes(b)
    cases["truncated scales"] = bytes(g[:20])
    b = bytearray(g); b[16:24] = np.float64(-1.0).tobytes(); cases["negative scale"] = bytes(b)
    b = bytearray(g); b[16:24] = np.float64(np.inf).tobytes(); cases["inf scale"] = bytes(b)
    cases["short payload"] = bytes(g[:-1])
    cases["trailing byte"] = bytes(g) + b"\x00"
    b = bytearray(g); b[24] = 0x13; cases["padding bit"] = bytes(b)  # bit 4 with cols = 4
    f = bytearray(b"APMM\x01\x00\x00\xff\x01\x00\x00\x00\x01\x00\x00\x00") + np.float32(1).tobytes()
    cases["float ok"] = bytes(f)
    f2 = bytearray(f); f2[6] = 1; cases["float with width"] = bytes(f2)
    f3 = bytearray(f); f3[7] = 0; cases["float with granularity"] = bytes(f3)
    return cases


def test_parse_errors_match_reference_classes(ap, reference):
    """Every corrupt image fails with the reference's error class: ParseError from
    parse_tensor, or OutOfRange for padding bits via to_packed -> PackedBitPlanes
    (bitplane.cpp:22-32). Quantized images go through the reference's parse_tensor +
    to_packed; float images through parse_tensor only (expected classes written out)."""
    from oracle import OracleError
    float_expect = {"float ok": None, "float with width": "ParseError",
                    "float with granularity": "ParseError"}
    for name, data in _corrupt_cases().items():
        ours = None
        try:
            t = ap.parse_tensor(data)
            if t.kind == ap.TensorKind.QuantizedBipolar:
                t.to_packed()
        except ap.Error as e:
            ours = type(e).__name__
        if name in float_expect:
            assert ours == float_expect[name], name
            continue
        theirs = None
        try:
            reference.parse_to_packed(data, 2, 1)
        except OracleError as e:
            theirs = e.name
        assert ours == theirs, (name, ours, theirs)
        assert ours is not None, name


def test_serialize_validation(ap):
    with pytest.raises(ap.OutOfRange):
        ap.serialize_tensor(ap.TensorFile(ap.TensorKind.QuantizedBipolar, 2, 0, 1, 4,
                                          np.array([0.0]), np.empty(0, np.float32),
                                          np.array([3, 5], np.uint32)))


def test_file_errors(ap, tmp_path):
    with pytest.raises(ap.IoError):
        ap.read_tensor_file(tmp_path / "missing.apmm")


@pytest.mark.gpu
def test_device_upload_equals_to_packed(gpu, golden, tmp_path):
    """apmm_cu_tensor_upload / apmm_tensor_file_load: the planes land in device memory in
    the PackedBitPlanes layout verbatim (== to_packed().words()), the scales bit-exact, a
    float tensor widened to f64 like to_real."""
    import torch
    ap, ctx = gpu
    for f in golden["tensor_files"]:
        path = os.path.join(GOLD, f["file"])
        t = ap.read_tensor_file(path)
        if f["kind"] == 1:
            planes, scales = t.cu_upload(ctx=ctx, stream=torch.cuda.current_stream())
            torch.cuda.synchronize()
            assert planes.cpu().numpy().view(np.uint32).tolist() == f["words"]
            assert [float(v).hex() for v in scales.cpu().numpy()] == f["scales"]
            t2, planes2, scales2 = ap.load_tensor_file(path)
            assert torch.equal(planes2.cpu(), planes.cpu()) and torch.equal(scales2.cpu(), scales.cpu())
            # the uploaded planes feed matmul_ap directly
            x = ap.PackedBitPlanes(f["rows"], f["cols"], ap.BitWidth(f["n"]),
                                   np.array(f["words"], np.uint32))
            assert np.array_equal(ap.matmul_ap(t.to_packed(), x, ctx=ap.Context(0)),
                                  ap.matmul_ap(x, x, ctx=ap.Context(0)))
        else:
            values = t.cu_upload(ctx=ctx, stream=torch.cuda.current_stream())
            torch.cuda.synchronize()
            assert [float(v).hex() for v in values.cpu().numpy().reshape(-1)] == f["values"]
            _, v2 = ap.load_tensor_file(path)
            assert torch.equal(v2.cpu(), values.cpu())
    # a big per-row W2 weight tensor written by the host serializer, uploaded, multiplied
    rng = np.random.default_rng(3)
    q = ap.quantize(rng.uniform(-1, 1, size=(300, 1000)), ap.BitWidth(2), ap.Granularity.PerRow,
                    ctx=ap.Context(0))
    tf = ap.TensorFile(ap.TensorKind.QuantizedBipolar, 2, 1, 300, 1000, q.scales,
                       np.empty(0, np.float32), q.packed.words())
    p = tmp_path / "w.apmm"
    p.write_bytes(ap.serialize_tensor(tf))
    _, planes, scales = ap.load_tensor_file(p)
    assert np.array_equal(planes.cpu().numpy().view(np.uint32), q.packed.words())
    assert np.array_equal(scales.cpu().numpy(), q.scales)
