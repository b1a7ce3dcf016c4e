"""B200-native CodeQuant Stage-4 path: the LUT-based quantized MoE expert matmul.

Host side mirrors the reference's operator API (reference pkg/src/codequant:
lutgemm.py, quant.py, kernels/__init__.py, and the MoE block of model.py);
every computation runs in libcq_b200.so (hand-written sm_100a CUDA, C ABI in
include/cq_b200.h).  No CPU fallback: without the library or a CUDA device,
the compute entry points raise.
"""

from .errors import (CodequantError, ConfigError, DivergenceError, FormatError,  # noqa: F401
                     ShapeError, SingularMatrixError, StageError)
from .lutgemm import (BENCH_HEADER, BenchRow, LUTile, PackedClusteredWeights,  # noqa: F401
                      bench_gemm, build_lut, lut_gemm, lut_gemm_tc, pack_weights, reference_gemm)
from .moe import ExpertStack, MoELayer, moe_layer  # noqa: F401
from .quant import (QuantizedActivations, QuantSpec, dequantize, fake_quant,  # noqa: F401
                    pack_nibbles, quantize_activations, unpack_nibbles)

__version__ = "0.1.0"
