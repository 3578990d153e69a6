"""paper_2104_05755_b200 — the Tensor Processing Primitives BRGEMM hot path,
B200-native (sm_100a).

Drop-in for the reference operator API of ``tensorprim``
(/root/reference/pkg/src/tensorprim/__init__.py:12-105) on the BRGEMM path:
same names, argument meaning, blocked layouts and exceptions; buffers are
CUDA tensors and every compute call runs a hand-written sm_100a kernel from
``libtpp_b200.so`` (C ABI: include/tpp_b200.h).  There is no CPU fallback.
"""

from .dtypes import COMPUTE_DTYPE, DType
from .tensor import (
    Bcast,
    SplitTensor,
    TensorDesc,
    TensorError,
    TensorView,
    alloc,
    alloc_bitmask,
    bits_of,
    bitmask_bytes,
    broadcast,
    convert,
    desc,
    from_array,
    mask_to_bool,
    pack_fp32,
    split_fp32,
    to_array,
    view_at,
)
from .ops import (
    Approx,
    BinaryKind,
    CmpOp,
    InvalidSpecError,
    Kernel,
    KernelSpec,
    PrngState,
    ReduceAxis,
    ReduceOp,
    ReduceSpec,
    TernaryKind,
    TransformKind,
    TransformSpec,
    UnaryKind,
    apply_binary,
    apply_ternary,
    apply_unary,
    dispatch,
    infer_output_desc,
    reduce,
    transform,
)
from .contraction import (
    ALayout,
    BlockingParams,
    BrgemmBatch,
    ComputePath,
    DEFAULT_BLOCKING,
    Engine,
    GemmSpec,
    GroupedBatch,
    brgemm,
    brgemm_grouped,
    gemm,
    matmul,
    spec_for_views,
    vnni_pack_a,
    vnni_unpack_a,
)
from .kernels import (
    Conv2d,
    ConvSpec,
    DilatedConvSpec,
    dilated_conv1d_forward,
    FcLayer,
    FcSpec,
    SoftmaxSpec,
    fc_forward,
    layernorm,
    layernorm_blocked,
    softmax,
    softmax_xent_blocked,
    split_sgd_flat,
    split_sgd_step,
)
from ._lib import TppUnavailableError
from . import parallel
from .training import BlockedMLP

__version__ = "0.1.0"
