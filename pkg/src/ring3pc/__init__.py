"""`ring3pc` -- the reference package's import path, served by the B200
implementation (north_star: keep the reference API in pkg/src so existing
programs are a drop-in).

Putting `pkg/src` on sys.path (or `pip install ./pkg`) makes

    import ring3pc
    from ring3pc import gates, verify, nonlinear, ppml
    from ring3pc.runtime import Session

resolve to `paper_2411_09287_b200`: every submodule of the reference
(reference pkg/src/ring3pc/{rings,prg,transport,sharing,runtime,gates,grvec,
verify,nonlinear,ppml,circuit,cli}.py) is registered under its `ring3pc.*`
name, so unmodified reference programs run on the GPU.  Share arrays are
CUDA int64 tensors (uint64 semantics); `ring3pc.host(t)` copies one to a
numpy uint64 array.
"""

from __future__ import annotations

import importlib
import os
import sys

__version__ = "0.1.0"

_REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if os.path.isdir(os.path.join(_REPO, "paper_2411_09287_b200")) and _REPO not in sys.path:
    sys.path.insert(0, _REPO)

_IMPL = "paper_2411_09287_b200"
SUBMODULES = ("rings", "prg", "transport", "sharing", "runtime", "gates", "grvec", "verify",
              "nonlinear", "ppml", "circuit", "cli")

for _name in SUBMODULES:
    _mod = importlib.import_module(f"{_IMPL}.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

from paper_2411_09287_b200 import (AbortError, AdversaryConfig, GrElem, GrModulus, Injection,  # noqa: E402,F401
                                   Party, Phase, Ring, RingElem, Session, device_array, host,
                                   modulus_for_degree)
