"""The maintainer-side ctypes binding shown in INTEGRATION.md §2
(integration/tensorprim_b200.py): its descriptor matches the header's
layout, it translates a reference GemmSpec exactly as this package does,
and (GPU) it computes the reference's bits through the C ABI."""

import ctypes as C
import os
import sys
import types

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "integration"))
import tensorprim_b200 as stub  # noqa: E402

from paper_2104_05755_b200 import _lib  # noqa: E402


def _ref_like_spec(m, n, k, beta=1.0, dt="fp32", vnni=False):
    """A duck-typed stand-in for tensorprim.GemmSpec (same field names and
    enum values as contraction.py:34-85, dtypes.py:17-24)."""
    E = lambda v: types.SimpleNamespace(value=v)  # noqa: E731
    acc = {"fp64": "fp64", "int8": "int32"}.get(dt, "fp32")
    return types.SimpleNamespace(m=m, n=n, k=k, lda=m, ldb=k, ldc=m, in_dtype=E(dt), out_dtype=E(acc),
                                 a_layout=E("vnni" if vnni else "plain"), compute_path=E("native"), beta=beta)


def test_descriptor_layout_matches_header_and_package():
    assert C.sizeof(stub.GemmDesc) == C.sizeof(_lib.GemmDescC)
    for (n1, _), (n2, _) in zip(stub.GemmDesc._fields_, _lib.GemmDescC._fields_):
        assert n1 == n2 and getattr(stub.GemmDesc, n1).offset == getattr(_lib.GemmDescC, n2).offset


def test_translation_equals_package_spec():
    import paper_2104_05755_b200 as tpp
    ref = _ref_like_spec(64, 32, 48, beta=0.5, dt="bf16", vnni=True)
    d = stub.desc_from_spec(ref, engine="ordered")
    ours = tpp.GemmSpec(64, 32, 48, 64, 48, 64, in_dtype=tpp.DType.BF16, out_dtype=tpp.DType.FP32, beta=0.5,
                        a_layout=tpp.ALayout.VNNI, engine=tpp.Engine.ORDERED).c()
    for name, _ in stub.GemmDesc._fields_:
        assert getattr(d, name) == getattr(ours, name), name


def test_translation_of_the_real_reference_spec():
    """With the reference importable (build container), translate its own GemmSpec."""
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, src)
    try:
        import tensorprim as tp
    except Exception as e:  # pragma: no cover
        pytest.skip(f"reference not importable: {e}")
    spec = tp.GemmSpec(16, 8, 32, 16, 32, 16, in_dtype=tp.DType.INT8, out_dtype=tp.DType.INT32, beta=1.0)
    d = stub.desc_from_spec(spec)
    assert (d.m, d.n, d.k, d.in_dtype, d.out_dtype, d.a_vnni, d.engine, d.beta) == (16, 8, 32, 5, 3, 0, 1, 1.0)


def test_library_loads_and_binds():
    lib = stub.load(_lib.LIB_PATH)
    assert lib.tpp_brgemm_stride.argtypes[0]._type_ is stub.GemmDesc


@pytest.mark.gpu
def test_stub_brgemm_bitwise_on_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import tpp_oracle as O
    lib = stub.load(_lib.LIB_PATH)
    rng = np.random.default_rng(5)
    m = n = k = 64
    cnt = 8
    a = rng.uniform(-1, 1, m * k * cnt).astype(np.float32)
    b = rng.uniform(-1, 1, k * n * cnt).astype(np.float32)
    c0 = rng.uniform(-1, 1, m * n).astype(np.float32)
    ad, bd, cd = (torch.from_numpy(v.copy()).cuda() for v in (a, b, c0))
    stub.brgemm_stride_device(lib, _ref_like_spec(m, n, k), ad.data_ptr(), bd.data_ptr(), m * k, k * n, cnt,
                              cd.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    want = O.brgemm([O.load_a(a, i * m * k, m, k, m, "fp32") for i in range(cnt)],
                    [O.load_b(b, i * k * n, k, n, k, "fp32") for i in range(cnt)], c0.reshape(n, m).T, beta=1.0)
    assert cd.cpu().numpy().tobytes() == want.T.reshape(-1).tobytes()
    bad = _ref_like_spec(m, n, k)
    bad.ldb = 3   # ldb < k: the reference raises TensorError before computing
    with pytest.raises(ValueError):
        stub.brgemm_stride_device(lib, bad, ad.data_ptr(), bd.data_ptr(), m * k, k * n, cnt, cd.data_ptr())
