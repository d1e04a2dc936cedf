"""B200-native LoRA-Switch hot path (arXiv 2405.17741).

The product is the C-ABI library ``liblsw.so`` (include/lsw.h) built from
``csrc/`` for sm_100a; this package is its thin Python binding plus the
host-side harness (model setup from ``synth``).  Importing it loads the
library and fails loudly if it has not been built -- there is no CPU path.
"""
from .binding import (  # noqa: F401
    LoraSwitch, LswError, KINDS, GROUPS, IMPL, lib, load_library, LIB_PATH, SYMBOLS,
)

lib()   # fail at import if liblsw.so is missing
