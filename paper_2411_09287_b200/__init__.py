"""ring3pc-b200: B200-native (sm_100a) data-parallel core of the arXiv
2411.09287 three-party honest-majority protocol suite.

Drop-in for the reference `ring3pc` package's API for the hot path (share
generation, Pi_mul/Pi_dot, Pi_trunc, GR batch verification, edaBits/ripple
ReLU): the same module names, classes and signatures, with share arrays held
as torch.int64 CUDA tensors (uint64 semantics) and every ring operation
executed by the hand-written kernels in libr3b200.so.  Use `host(t)` to get
a numpy uint64 copy.  A user of `ring3pc` can alias the package:

    import sys, paper_2411_09287_b200 as ring3pc
    sys.modules["ring3pc"] = ring3pc
"""

__version__ = "0.1.0"

from .rings import GrElem, GrModulus, RingElem, modulus_for_degree  # noqa: F401
from .transport import AbortError, AdversaryConfig, Injection, Phase  # noqa: F401
from .sharing import Ring  # noqa: F401
from .runtime import Party, Session  # noqa: F401
from ._lib import to_host as host, to_device as device_array  # noqa: F401
