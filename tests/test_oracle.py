"""Pins the plain-C oracle (oracle/apmm_oracle.c) to the reference: the known-answer
vectors of the reference's own tests (proj/tests/*.cpp, cited per test), the golden
fixture produced by running the reference (tests/golden, oracle/gen_golden.py), and --
when oracle/_ref is built -- the reference library itself on random inputs."""
import numpy as np
import pytest

from oracle import PER_ROW, PER_TENSOR, OracleError


def test_mt19937_64_standard_value(oracle):
    # C++ [rand.predef]: the 10000th draw of a default-constructed mt19937_64 (seed 5489).
    assert int(oracle.rng(5489).next_u64(10000)[-1]) == 9981545732273789042


def test_rng_matches_golden(oracle, golden):
    for seed, draws in golden["rng"].items():
        assert [str(int(v)) for v in oracle.rng(int(seed)).next_u64(len(draws))] == draws


def test_decode_tables(oracle):
    # test_bipolar.cpp:10-36
    assert [oracle.lib.orc_decode(c, 2) for c in range(4)] == [-3, -1, 1, 3]
    assert [oracle.lib.orc_decode(c, 1) for c in range(2)] == [-1, 1]
    assert oracle.lib.orc_decode(0b101, 3) == 3
    for n in range(1, 9):
        for c in range(1 << n):
            assert oracle.lib.orc_decode(c, n) == 2 * c - ((1 << n) - 1)


def test_quantize_known_answers(oracle):
    # test_bipolar.cpp:111-156
    codes, s = oracle.quantize(np.array([[3.0, -1.0, 1.0, -3.0]]), 2, PER_TENSOR)
    assert s[0] == 1.0 and oracle.decode(codes, 2).tolist() == [[3, -1, 1, -3]]
    codes, s = oracle.quantize(np.array([[0.0]]), 2, PER_TENSOR)
    assert s[0] == 1.0 and oracle.decode(codes, 2).tolist() == [[1]]
    codes, s = oracle.quantize(np.array([[2.0, -2.0, 0.5, 0.0]]), 2, PER_TENSOR)
    assert s[0] == pytest.approx(2.0 / 3.0) and oracle.decode(codes, 2).tolist() == [[3, -3, 1, 1]]
    codes, s = oracle.quantize(np.array([[3.0, -3.0], [30.0, -30.0]]), 2, PER_ROW)
    assert s.tolist() == [1.0, 10.0] and oracle.decode(codes, 2)[:, 0].tolist() == [3, 3]
    codes, s = oracle.quantize(np.array([[0.0, 0.0], [5.0, -5.0]]), 3, PER_ROW)
    assert s[0] == 1.0 and oracle.decode(codes, 3)[0].tolist() == [1, 1]
    assert s[1] == pytest.approx(5.0 / 7.0)
    with pytest.raises(OracleError):
        oracle.quantize(np.array([[1.0, np.nan]]), 2, PER_TENSOR)
    with pytest.raises(OracleError):
        oracle.quantize(np.array([[np.inf]]), 4, PER_TENSOR)


def test_quantize_matches_golden_bit_exact(oracle, golden):
    for case in golden["quantize"]:
        x = np.array([float.fromhex(h) for h in case["x"]]).reshape(case["rows"], case["cols"])
        codes, scales = oracle.quantize(x, case["n"], case["gran"])
        assert codes.reshape(-1).tolist() == case["codes"]
        assert [float(v).hex() for v in scales] == case["scales"]


def test_pack_known_answers(oracle):
    # test_bitplane.cpp:19-50
    assert oracle.pack(np.array([[1]], np.uint8), 1).tolist() == [0x1]
    assert oracle.pack(np.ones((1, 33), np.uint8), 1).tolist() == [0xFFFFFFFF, 0x1]
    codes = np.array([[0b11, 0b10], [0b01, 0b00]], np.uint8)  # values [[3,1],[-1,-3]]
    assert oracle.pack(codes, 2).tolist() == [0b01, 0b01, 0b11, 0b00]


def test_pack_matches_golden_and_round_trips(oracle, golden):
    for case in golden["pack"]:
        codes = np.array(case["codes"], np.uint8).reshape(case["rows"], case["cols"])
        words = oracle.pack(codes, case["n"])
        assert words.tolist() == case["words"]
        assert np.array_equal(oracle.unpack(words, case["rows"], case["cols"], case["n"]), codes)
        assert oracle.check_padding(words, case["rows"], case["cols"], case["n"]) == 0


def test_padding_validation(oracle):
    # test_bitplane.cpp:138-143: bit 1 is padding when K = 1
    assert oracle.check_padding(np.array([0x2], np.uint32), 1, 1, 1) == 2
    assert oracle.check_padding(np.array([0x1], np.uint32), 1, 1, 1) == 0


def test_dot_known_answers(oracle):
    # test_kernel.cpp:22-56
    a = np.array([0xA5A5A5A5], np.uint32)
    assert oracle.dot_1bit_xor(a, a, 32) == 32
    assert oracle.dot_1bit_xor(np.array([0xFFFFFFFF], np.uint32), np.array([0], np.uint32), 32) == -32
    assert oracle.dot_1bit_xor(np.array([0b1100], np.uint32), np.array([0b1010], np.uint32), 4) == 0
    a = np.array([0xFFFFFFFF] * 3 + [0xF], np.uint32)
    b = a.copy()
    assert oracle.dot_1bit_xor(a, b, 100) == 100
    b[1] = 0
    assert oracle.dot_1bit_xor(a, b, 100) == 100 - 64
    with pytest.raises(OracleError):
        oracle.dot_1bit_xor(np.zeros(1, np.uint32), np.zeros(2, np.uint32), 32)
    with pytest.raises(OracleError):
        oracle.dot_1bit_xor(np.zeros(1, np.uint32), np.zeros(1, np.uint32), 0)


def test_worked_two_bit_example(oracle, golden):
    # test_kernel.cpp:125-136 / acceptance.cpp:81-106: planes (0,-2,2,0) recover to 0
    case = golden["plane_products"][0]
    wc = np.array(case["w_codes"], np.uint8).reshape(1, 2)
    xc = np.array(case["x_codes"], np.uint8).reshape(1, 2)
    stack = oracle.plane_products(oracle.pack(wc, 2), 1, 2, oracle.pack(xc, 2), 1, 2, 2)
    assert stack.reshape(-1).tolist() == case["stack"] == [0, -2, 2, 0]
    assert oracle.recover(stack).reshape(-1).tolist() == case["y"] == [0]
    assert oracle.matmul_ap(oracle.pack(wc, 2), 1, 2, oracle.pack(xc, 2), 1, 2, 2).tolist() == [[0]]


def test_overflow_bound(oracle):
    # test_kernel.cpp:183-200, verify.cpp:373-409
    assert oracle.overflow_bound(1, 1, 4096) == 4096
    assert oracle.overflow_bound(3, 4, 10752) == 1128960
    assert oracle.overflow_bound(8, 8, 33025) <= 2**31 - 1 < oracle.overflow_bound(8, 8, 33026)
    w = np.zeros(8 * ((33026 + 31) // 32), np.uint32)
    with pytest.raises(OracleError) as e:
        oracle.matmul_ap(w, 1, 8, w, 1, 8, 33026)
    assert e.value.name == "OverflowBound"


def test_matmul_matches_golden(oracle, golden):
    for c in golden["matmul"]:
        w = np.array(c["w_words"], np.uint32)
        x = np.array(c["x_words"], np.uint32)
        y = oracle.matmul_ap(w, c["rows_w"], c["n_w"], x, c["rows_x"], c["n_x"], c["k"])
        assert y.reshape(-1).tolist() == c["y"], c


def test_randomized_corpus_and_schedule_independence(oracle):
    # test_kernel.cpp:208-245: any TileConfig == stack+recover == decoded oracle
    rng = oracle.rng(31)
    for _ in range(100):
        m, n, k = rng.range(1, 32), rng.range(1, 32), rng.range(1, 200)
        nw, nx = rng.range(1, 8), rng.range(1, 8)
        wc, xc = rng.random_codes(m, k, nw), rng.random_codes(n, k, nx)
        wp, xp = oracle.pack(wc, nw), oracle.pack(xc, nx)
        want = oracle.decoded_matmul(wc, nw, xc, nx)
        for tile in [(64, 64, 512), (1, 1, 32), (m + 5, n + 5, 64), (3, 2, 96)]:
            assert np.array_equal(oracle.matmul_ap(wp, m, nw, xp, n, nx, k, tile), want)
        if nw <= 4 and nx <= 4:
            assert np.array_equal(oracle.recover(oracle.plane_products(wp, m, nw, xp, n, nx, k)), want)
        assert np.array_equal(oracle.matmul_ap_mt(wp, m, nw, xp, n, nx, k, 3), want)


def test_dequant_worked_example(oracle):
    # test_cli.cpp:147-181: quantize [3,1] and [-1,3] at 2 bits, matmul --dequant -> 0
    wc, ws = oracle.quantize(np.array([[3.0, 1.0]]), 2, PER_TENSOR)
    xc, xs = oracle.quantize(np.array([[-1.0, 3.0]]), 2, PER_TENSOR)
    y = oracle.matmul_ap(oracle.pack(wc, 2), 1, 2, oracle.pack(xc, 2), 1, 2, 2)
    assert oracle.dequant_epilogue(y, ws, PER_TENSOR, xs, PER_TENSOR).tolist() == [[0.0]]


def test_oracle_equals_reference_library(oracle, reference):
    rng = oracle.rng(7)
    for _ in range(60):
        m, n, k = rng.range(1, 40), rng.range(1, 40), rng.range(1, 400)
        nw, nx = rng.range(1, 8), rng.range(1, 8)
        wc, xc = rng.random_codes(m, k, nw), rng.random_codes(n, k, nx)
        wp, xp = oracle.pack(wc, nw), oracle.pack(xc, nx)
        assert np.array_equal(wp, reference.pack(wc, nw))
        assert np.array_equal(oracle.matmul_ap(wp, m, nw, xp, n, nx, k),
                              reference.matmul_ap(wp, m, nw, xp, n, nx, k))
        x = np.random.default_rng(m * 1000 + k).uniform(-50, 50, size=(m, k))
        for gran in (PER_TENSOR, PER_ROW):
            c1, s1 = oracle.quantize(x, nw, gran)
            c2, s2 = reference.quantize(x, nw, gran)
            assert np.array_equal(c1, c2) and np.array_equal(s1, s2)


def test_reference_run_verify_passes(reference):
    passed, detail = reference.run_verify(seed=1, cases=200)
    assert len(passed) == 9 and all(passed), detail
