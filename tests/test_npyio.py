"""Real-model tensor ingestion: strict npy v1.0 f32 I/O and dump trees
(reference ``npyio.py:22-77``, ``harness/dump.py:19-82``; behaviour pinned
by the reference's ``tests/test_npyio.py`` / ``tests/test_dump.py`` cases:
round trips, numpy interoperability, each malformed field rejected with
``FormatError``, shape drift -> ``ContractError``)."""

import struct

import numpy as np
import pytest

from paper_2604_18348_b200.errors import ContractError, FormatError
from paper_2604_18348_b200.npyio import ingest_dump, read_npy, write_dump, write_npy


@pytest.mark.parametrize("shape", [(0,), (7,), (3, 5), (2, 3, 4)])
def test_round_trip_and_numpy_interop(tmp_path, shape):
    a = np.random.default_rng(1).normal(size=shape).astype(np.float32)
    p = tmp_path / "a.npy"
    write_npy(p, a)
    assert (10 + struct.unpack("<H", p.read_bytes()[8:10])[0]) % 64 == 0
    b = read_npy(p)
    assert b.dtype == np.float32 and b.shape == a.shape and np.array_equal(a, b)
    assert np.array_equal(np.load(p), a)
    np.save(tmp_path / "n.npy", a)
    assert np.array_equal(read_npy(tmp_path / "n.npy"), a)


def _corrupt(tmp_path, mutate):
    p = tmp_path / "x.npy"
    write_npy(p, np.ones((4, 2), np.float32))
    raw = bytearray(p.read_bytes())
    p.write_bytes(bytes(mutate(raw)))
    return p


@pytest.mark.parametrize("case", ["magic", "version", "descr", "fortran", "shape", "payload",
                                  "header", "missing"])
def test_rejects_malformed(tmp_path, case):
    def edit_header(raw, old, new):
        return raw.replace(old, new.ljust(len(old)))
    mut = {
        "magic": lambda r: b"\x00" + r[1:],
        "version": lambda r: r[:6] + bytes((2, 0)) + r[8:],
        "descr": lambda r: edit_header(r, b"'<f4'", b"'<f8'"),
        "fortran": lambda r: edit_header(r, b"False", b"True"),
        "shape": lambda r: edit_header(r, b"(4, 2)", b"(4,-2)"),
        "payload": lambda r: r[:-4],
        "header": lambda r: edit_header(r, b"{'descr'", b"['descr'"),
        "missing": lambda r: edit_header(r, b"'fortran_order': False, ", b""),
    }[case]
    with pytest.raises(FormatError):
        read_npy(_corrupt(tmp_path, mut))


def test_rejects_non_f32(tmp_path):
    np.save(tmp_path / "f64.npy", np.ones(3))
    with pytest.raises(FormatError):
        read_npy(tmp_path / "f64.npy")
    np.save(tmp_path / "fo.npy", np.asfortranarray(np.ones((3, 2), np.float32)))
    with pytest.raises(FormatError):
        read_npy(tmp_path / "fo.npy")


def _inputs(steps=2, layers=2, heads=3, L=17, D=8, seed=0):
    rng = np.random.default_rng(seed)
    return [[[tuple(rng.normal(size=(L, D)).astype(np.float32) for _ in range(3))
              for _ in range(heads)] for _ in range(layers)] for _ in range(steps)]


def test_dump_round_trip(tmp_path):
    x = _inputs()
    write_dump(tmp_path, x)
    y = ingest_dump(tmp_path)
    for t in range(2):
        for l in range(2):
            for h in range(3):
                for a, b in zip(x[t][l][h], y[t][l][h]):
                    assert np.array_equal(a, b)


def test_dump_errors(tmp_path):
    x = _inputs(steps=2, layers=1, heads=2)
    write_dump(tmp_path / "ok", x)
    # non-contiguous head indices
    (tmp_path / "ok" / "step0" / "layer0" / "head1").rename(tmp_path / "ok" / "step0" / "layer0" / "head5")
    with pytest.raises(FormatError):
        ingest_dump(tmp_path / "ok")
    # shape drift between steps
    y = _inputs(steps=2, layers=1, heads=2)
    y[1][0][1] = tuple(np.zeros((9, 8), np.float32) for _ in range(3))
    write_dump(tmp_path / "drift", y)
    with pytest.raises(ContractError):
        ingest_dump(tmp_path / "drift")
    # inconsistent q/k/v
    z = _inputs(steps=1, layers=1, heads=1)
    q, k, v = z[0][0][0]
    z[0][0][0] = (q, k, v[:5])
    write_dump(tmp_path / "qkv", z)
    with pytest.raises(ContractError):
        ingest_dump(tmp_path / "qkv")
    # rank and missing files
    write_dump(tmp_path / "rank", _inputs(steps=1, layers=1, heads=1))
    write_npy(tmp_path / "rank" / "step0" / "layer0" / "head0" / "q.npy", np.ones(4, np.float32))
    with pytest.raises(FormatError):
        ingest_dump(tmp_path / "rank")
    (tmp_path / "rank" / "step0" / "layer0" / "head0" / "q.npy").unlink()
    with pytest.raises(FormatError):
        ingest_dump(tmp_path / "rank")
    with pytest.raises(FormatError):
        ingest_dump(tmp_path / "nope")


@pytest.mark.gpu
def test_load_layer_drives_the_layer_step(gpu, tmp_path):
    """A dumped layer loaded through the pinned staging path gives the same
    device tensors (bf16) and the same layer output as the in-memory inputs."""
    import torch
    from paper_2604_18348_b200.npyio import load_layer
    from workload.synthetic import CRIT7_SPEC, gen_synthetic
    H, L, D = 2, 3000, 64
    steps = [[[tuple(a) for a in (gen_synthetic(CRIT7_SPEC, L, D, 1, 1, 10 + h)[0][0] for h in range(H))]]]
    write_dump(tmp_path, steps)
    Q, K, V = load_layer(tmp_path, 0, 0)
    ref = [torch.stack([torch.from_numpy(steps[0][0][h][i]) for h in range(H)]).bfloat16().cuda()
           for i in range(3)]
    for a, b in zip((Q, K, V), ref):
        assert a.dtype == torch.bfloat16 and torch.equal(a, b)
    p = gpu.PipelineParams(q_clusters=65, topk=25, full_layer_quota=0.0)
    o1 = gpu.LayerSession(p, out_dtype=torch.float32).step(Q, K, V).clone()
    o2 = gpu.LayerSession(p, out_dtype=torch.float32).step(*ref).clone()
    assert torch.equal(o1, o2)


def test_zero_element_arrays_round_trip(tmp_path):
    """Valid zero-element arrays (e.g. shape (0, 64)) read back as empty arrays."""
    from paper_2604_18348_b200.npyio import read_npy, write_npy
    for shape in [(0, 64), (0,), (3, 0)]:
        p = tmp_path / f"z{len(shape)}_{shape[0]}.npy"
        write_npy(p, np.zeros(shape, np.float32))
        out = read_npy(p)
        assert out.shape == shape and out.dtype == np.float32
        assert np.load(p).shape == shape
