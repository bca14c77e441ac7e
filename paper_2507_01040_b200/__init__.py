"""B200-native (sm_100a) Clifford convolution / multivector activation /
basic-block inference: a drop-in for the layer API of the reference
`mvkernels` package (arXiv 2507.01040), backed by libclifford_b200.so
(C-ABI: include/clifford_b200.h), called through its PyTorch operator
registration torch.ops.clifford_b200.* (csrc_torch/clifford_ops.cpp)."""

from .activation import (ActivationConfig, AggMode, activation_flops, activation_forward, gate_preactivation,
                         gather_vpack, make_activation_config, sigmoid)
from .algebra import (BladeProductTable, Signature, all_valid_signatures, blade_product, cayley_tensor,
                      geometric_product, product_table, schedule_flop_count, schedule_terms, validate_signature)
from .block import BasicBlock, block_forward, make_basic_block
from .conv import ConvLayer, build_expanded_kernel, conv_flops, conv_forward, make_conv_layer
from .layout import Dims, LayoutTag, gather_index_table, read_tensor, spatial_coords, write_tensor
from .specialize import FmaTerm, OpSchedule, build_schedule, schedule_for
from .linear import LinearLayer, linear_flops, linear_forward, make_linear_layer
from .metrics import max_abs_error, max_rel_error
from ._ops import launch_count
from . import errors

__version__ = "0.2.0"
