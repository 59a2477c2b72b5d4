"""B200-native QEFT structured mixed-precision linear layer (arXiv 2410.08661).

Drop-in for the reference package's hot path (`qeft.quantizer`, `qeft.kernels`,
`qeft.tuning`): the same Python names and argument meaning, with the compute
running in hand-written sm_100a CUDA kernels behind a C ABI
(include/qeft_b200.h, libqeft_b200.so).
"""

__version__ = "0.1.0"
