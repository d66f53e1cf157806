"""B200-native census template-matching stereo ranger (arxiv 2604.07980 hot path).

The compute lives in paper_2604_07980_b200/lib/libranger_cuda.so (sm_100a
kernels + the C ABI of include/ranger_cuda.h); this package is the Python
mirror of the reference's API (`ranger`), the synthetic frame source
(`synth`) and the batched throughput engine (`engine`).
"""
from . import ranger  # noqa: F401
