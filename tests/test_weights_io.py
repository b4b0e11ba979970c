"""PBKD weight files (reference weights_io.cpp:68-319,
test_weights_io.cpp): the product's writer / reader against the reference
library itself (oracle/_ref), byte for byte.  CPU only."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import paper_2012_03096_b200 as P
from tests.conftest import spec_text


def _ref_save(ref, spec, seed, k, kind, cand_seed, path):
    """Reference: teacher init_weights(seed), block k (0: none) replaced by
    build_candidate(kind, ..., cand_seed) named like the teacher block
    (reassemble, distill.cpp:319), save_weights(arrays_from_network)."""
    f = ref.fn("save_network_file", C.c_int, [C.c_char_p, C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.c_char_p])
    ref._check(f(spec.encode(), seed, k, kind, cand_seed, os.fsencode(path)))


def _ref_rebuild_kinds(ref, spec, path):
    nb = P.spec_num_blocks(spec)
    kinds = (C.c_int * nb)()
    h = C.c_uint64()
    f = ref.fn("rebuild_network_file", C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_uint64), C.c_void_p, C.c_int])
    ref._check(f(spec.encode(), os.fsencode(path), C.byref(h), C.cast(kinds, C.c_void_p), nb))
    return list(kinds)


def _ref_file_hash(ref, path):
    h = C.c_uint64()
    ref._check(ref.fn("file_hash", C.c_int, [C.c_char_p, C.POINTER(C.c_uint64)])(os.fsencode(path), C.byref(h)))
    return h.value


def _block_dims(spec, k):
    """(c_in, c_out, stride) of teacher block k (1-based) from the spec JSON."""
    s = json.loads(spec)
    c = s["input_shape"][0]
    for i, b in enumerate(s["blocks"], 1):
        if i == k:
            return c, b["out_channels"], b.get("stride", 1)
        c = b["out_channels"]
    raise IndexError(k)


@pytest.mark.parametrize("name", ["toy_teacher", "c1_small_vgg", "resnet18_cifar"])
def test_student_file_byte_identical(orc, ref, tmp_path, name):
    """A teacher with block 2 replaced by each candidate kind: the product's
    file equals the reference's byte for byte, and the file hashes agree."""
    spec = spec_text(name)
    tw = orc.teacher_init(spec, 31)
    for kind in range(4):
        blk = P.build_candidate(kind, *_block_dims(spec, 2), P.mix_seed(7, kind))
        ours, theirs = tmp_path / f"ours_{kind}.pbkd", tmp_path / f"ref_{kind}.pbkd"
        P.save_student_network(spec, tw, 2, kind, blk, ours)
        _ref_save(ref, spec, 31, 2, kind, P.mix_seed(7, kind), theirs)
        assert ours.read_bytes() == theirs.read_bytes()
        assert P.file_hash(ours) == _ref_file_hash(ref, theirs)


def test_rebuild_matches_reference(orc, ref, tmp_path):
    """rebuild_network_from_arrays on reference-written student files: the same
    block kinds as the reference's rebuild, and the rebuilt network's arrays
    are the file's (teacher blocks + the candidate's weights)."""
    spec = spec_text("c1_small_vgg")
    tw = orc.teacher_init(spec, 5)
    for kind in range(4):
        path = tmp_path / f"s{kind}.pbkd"
        _ref_save(ref, spec, 5, 3, kind, 99, path)
        kinds, flat = P.load_network_file(spec, path)
        assert list(kinds) == _ref_rebuild_kinds(ref, spec, path)
        assert kinds[2] == 1 + kind and not kinds[0] and not kinds[1] and not kinds[3]
        # rebuilt arrays = teacher blocks 1-2, the candidate, teacher block 4 + classifier
        blk = P.build_candidate(kind, *_block_dims(spec, 3), 99)
        again = tmp_path / f"again{kind}.pbkd"
        P.save_student_network(spec, tw, 3, kind, blk, again)
        assert again.read_bytes() == path.read_bytes()
        # the candidate's weights are part of the rebuilt network's arrays
        assert _contains(flat, blk)


def _contains(hay, needle):
    for i in np.flatnonzero(hay[:hay.size - needle.size + 1] == needle[0]):
        if np.array_equal(hay[i:i + needle.size], needle):
            return True
    return False


def test_teacher_round_trip_and_validation(orc, ref, tmp_path):
    spec = spec_text("toy_teacher")
    path = tmp_path / "t.pbkd"
    _ref_save(ref, spec, 123, 0, 0, 0, path)
    kinds, flat = P.load_network_file(spec, path)
    assert not any(kinds)
    assert np.array_equal(flat, orc.teacher_init(spec, 123))
    raw = path.read_bytes()
    bad = tmp_path / "bad.pbkd"
    bad.write_bytes(raw[:-3])
    with pytest.raises(P.WeightsError, match="truncated"):
        P.load_network_file(spec, bad)
    bad.write_bytes(b"NOPE" + raw[4:])
    with pytest.raises(P.WeightsError, match="bad magic"):
        P.load_network_file(spec, bad)
    bad.write_bytes(raw + b"\0")
    with pytest.raises(P.WeightsError, match="trailing"):
        P.load_network_file(spec, bad)
    with pytest.raises(P.WeightsError):  # arrays of another network
        P.load_network_file(spec_text("c1_small_vgg"), path)


@pytest.mark.gpu
def test_teacher_file_through_context(orc, ref, tmp_path):
    """Context.teacher_save_file writes the reference's file for the same
    teacher; teacher_load_file reads it back into the engine."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    spec = spec_text("c1_small_vgg")
    ctx = P.Context(0)
    ctx.teacher_init(spec, 77)
    ours, theirs = tmp_path / "ours.pbkd", tmp_path / "ref.pbkd"
    ctx.teacher_save_file(ours)
    _ref_save(ref, spec, 77, 0, 0, 0, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    ctx2 = P.Context(0)
    ctx2.teacher_load_file(spec, theirs)
    n = P.spec_num_floats(spec)
    assert np.array_equal(ctx2.teacher_weights(n), orc.teacher_init(spec, 77))
