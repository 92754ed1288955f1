"""CPU tests of the product's host side (libpbbgpu.so host C++ + the Python mirror).
No GPU compute is called here."""
import os
import random

import numpy as np
import pytest

import paper_2012_09511_b200 as pbb
from paper_2012_09511_b200 import _lib
from paper_2012_09511_b200.factoradic import compare, from_decimal, midpoint, to_decimal
from tests import golden_io


def test_taillard_matches_reference():
    for name, mat in golden_io.ref_instances().items():
        inst = pbb.taillard_named(name)
        assert np.array_equal(inst.p, mat), name


def test_generate_taillard_errors():
    with pytest.raises(ValueError):
        pbb.generate_taillard(20, 5, 0)          # seed 0 -> error (SPEC.md generate_taillard)
    with pytest.raises(ValueError):
        pbb.taillard_named("ta121")
    a = pbb.generate_taillard(20, 5, 873654221)
    assert np.array_equal(a.p, pbb.taillard_named("ta001").p)


def test_makespan_spec_examples():
    inst = pbb.Instance(2, 2, [[2, 3], [4, 1]])
    assert pbb.makespan(inst, [0, 1]) == 7
    assert pbb.makespan(inst, [1, 0]) == 9
    with pytest.raises(ValueError):
        pbb.makespan(inst, [0, 0])


def test_parse_instance_layouts():
    a = pbb.parse_instance("2 2\n2 3\n4 1")
    assert a.p.tolist() == [[2, 3], [4, 1]]
    b = pbb.parse_instance("2 2\n2 4\n3 1", machine_major=True)
    assert b.p.tolist() == [[2, 3], [4, 1]]
    with pytest.raises(ValueError):
        pbb.parse_instance("2 2\n1 2\n3 4\n5 6")


def test_neh_matches_reference():
    for key, ref in golden_io.ref_counts().items():
        if key.startswith("neh:"):
            s = pbb.neh(pbb.taillard_named(key[4:]))
            assert s.cmax == ref["cmax"] and s.perm == ref["perm"], key


# ---- factoradic boundary (test_factoradic.cpp:43-133) --------------------------------------------

def test_to_decimal_vectors():
    assert to_decimal([0, 0, 0, 0]) == 0
    assert to_decimal([2, 1, 1, 0]) == 15
    assert to_decimal([3, 2, 1, 0]) == 23
    with pytest.raises(ValueError):
        to_decimal([4, 0, 0, 0])
    with pytest.raises(ValueError):
        to_decimal([0, 0, 0, 1])


def test_from_decimal_bijection_8fact():
    assert from_decimal(15, 4) == [2, 1, 1, 0]
    with pytest.raises(ValueError):
        from_decimal(24, 4)
    for x in range(40320):
        assert to_decimal(from_decimal(x, 8)) == x


def test_compare_matches_decimal_order():
    rng = random.Random(11)
    for _ in range(2000):
        n = rng.randint(2, 10)
        fact = 1
        for k in range(2, n + 1):
            fact *= k
        xa, xb = rng.randrange(fact), rng.randrange(fact)
        assert compare(from_decimal(xa, n), from_decimal(xb, n)) == (xa > xb) - (xa < xb)


def test_midpoint_vectors():
    assert midpoint([0, 0, 0, 0], None) == [2, 0, 0, 0]
    assert to_decimal(midpoint([0, 0], None)) == 1
    rng = random.Random(42)
    for _ in range(3000):
        n = rng.randint(2, 9)
        fact = 1
        for k in range(2, n + 1):
            fact *= k
        a, b = rng.randrange(fact), rng.randrange(fact + 1)
        if a == b:
            continue
        a, b = min(a, b), max(a, b)
        m = midpoint(from_decimal(a, n), from_decimal(b, n) if b < fact else None)
        assert to_decimal(m) == (a + b) // 2
    rng = random.Random(43)
    for _ in range(1000):
        a, b = rng.randrange(5040), rng.randrange(5040)
        if a + 2 > b:
            continue
        mid = to_decimal(midpoint(from_decimal(a, 7), from_decimal(b, 7)))
        assert abs((mid - a) - (b - mid)) <= 1 and mid - a >= 1 and b - mid >= 1


def test_big_factoradic_roundtrip():
    import math
    n = 500
    for x in (0, 1, math.factorial(n) - 1, math.factorial(n) // 3):
        assert to_decimal(from_decimal(x, n)) == x


def test_normalize():
    assert pbb.normalize([(5, 9), (0, 3), (2, 4), (9, 9), (9, 12)]) == [(0, 4), (5, 9), (9, 12)]
    with pytest.raises(ValueError):
        pbb.normalize([(3, 1)])


def test_pool_without_gpu_fails_loudly():
    if _lib.load().pbbgpu_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(_lib.PbbError) as e:
        pbb.GpuPool(pbb.taillard_named("ta001"))
    assert e.value.code == _lib.PBBGPU_ERR_CUDA


def test_insertion_local_search_matches_reference():
    """Host insertion LS (seeded mt19937_64 tie-breaking) is bit-exact with the reference's."""
    for key, ref in golden_io.ref_counts().items():
        if not key.startswith("ils:"):
            continue
        inst = pbb.taillard_named(key[4:])
        s = pbb.insertion_local_search(inst, pbb.neh(inst), max_iterations=ref["iterations"], rng_seed=ref["rng_seed"])
        assert s.cmax == ref["cmax"] and s.perm == ref["perm"], key
        assert pbb.makespan(inst, s.perm) == s.cmax


def test_insertion_local_search_needs_a_budget():
    inst = pbb.taillard_named("ta001")
    with pytest.raises(ValueError):
        pbb.insertion_local_search(inst, pbb.neh(inst))


def test_checkpoint_format_matches_reference(tmp_path):
    """Our writer reproduces the reference's checkpoint_save bytes; its file loads back."""
    from math import factorial

    from paper_2012_09511_b200 import checkpoint as ck

    inst = pbb.taillard_named("ta021")
    ref_path = os.path.join(golden_io.GOLDEN, "ref_checkpoint_ta021.ckpt")
    d = ck.checkpoint_load(ref_path, inst)
    s = pbb.neh(inst)
    nf = factorial(20)
    assert d.best_value == s.cmax and d.best_schedule == s.perm and d.total_nodes == 123456789
    assert [(u.kmax, u.intervals) for u in d.units] == [(4, [(0, 1000), (5000, nf)]), (2, [(nf // 2, nf // 2 + 7)])]
    out = tmp_path / "mine.ckpt"
    ck.checkpoint_save(str(out), inst, d)
    assert out.read_bytes() == open(ref_path, "rb").read()
    with pytest.raises(ValueError):
        ck.checkpoint_load(ref_path, pbb.taillard_named("ta022"))  # different instance


def test_instance_fingerprint():
    from paper_2012_09511_b200 import checkpoint as ck

    assert f"{ck.instance_fingerprint(pbb.taillard_named('ta021')):016x}" == "23f4aba7591455ec"


# ---------------------------------------------------------------- wire protocol

def _ref_frames():
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_frames.txt")
    out = []
    for line in open(path):
        who, n, hx = line.split()
        out.append((who == "W", int(n), bytes.fromhex(hx)))
    return out


def test_wire_codec_reencodes_reference_frames_byte_for_byte():
    """Every frame the reference's encode() produced (tests/golden/ref_frames.txt: WORK requests
    and replies with intervals of [0, n!) for n = 5 .. 500, BEST / END with and without
    schedules) decodes and re-encodes to the same bytes, also with the interval endpoints passed
    through the pool boundary's factoradic digit vectors."""
    frames = _ref_frames()
    assert len(frames) >= 20
    for worker, n, fr in frames:
        assert pbb.wire_reencode(fr, worker) == fr
        assert pbb.wire_reencode(fr, worker, n) == fr


def test_wire_codec_rejects_malformed_frames():
    from paper_2012_09511_b200 import _lib

    worker, n, fr = _ref_frames()[0]
    with pytest.raises(_lib.PbbError):
        pbb.wire_reencode(fr[:-1], worker)                        # truncated
    with pytest.raises(_lib.PbbError):
        pbb.wire_reencode(fr + b"\x00", worker)                   # length mismatch
    bad = bytearray(fr)
    bad[4] = 9
    with pytest.raises(_lib.PbbError):
        pbb.wire_reencode(bytes(bad), worker)                     # unknown tag
    one = bytes.fromhex("0000000b0100000001000101000101")           # WORK reply [1, 1): a >= b
    with pytest.raises(_lib.PbbError):
        pbb.wire_reencode(one, False)
