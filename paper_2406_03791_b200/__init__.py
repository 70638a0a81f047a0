"""B200-native RNN-T / TDT greedy decoder (arXiv 2406.03791) behind the
reference rnnt-sim decoder interface.  CUDA kernels + C ABI live in csrc/
and build into librnntg.so; this package is the host-side mirror."""
from . import errors  # noqa: F401
from .decoders import (CapturedDecoder, DecodeAlgo, Exec, Hypothesis, Model, ModelDims,  # noqa: F401
                       build_decode_graph, decode_joint_evals, greedy_decode_sync_free,
                       label_looping_decode, replay_decode, tdt_label_looping_decode)
