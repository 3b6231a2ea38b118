"""paper_2605_19049_b200 — KV-buffered Gated DeltaNet decode on NVIDIA B200.

B200-native (sm_100a) implementation of the IO-aware serving mechanism of
arxiv 2605.19049 for Gated DeltaNet linear attention: buffered chunkwise
decode, tensor-core flush, parallel draft verification with accepted-prefix
commit, direct (KV-only) short-context decode, and the conventional recurrent
kernels as the in-run baseline.  The product is the C-ABI library
``liblabuf.so`` (include/la.h); :mod:`.labuf` is its thin ctypes binding.
"""
from .labuf import (LA_DT_BF16, LA_DT_F16, LA_DT_F32, LA_FLUSH_FORCE, LA_FLUSH_FULL,  # noqa: F401
                    LA_MODE_CHUNKWISE, LA_MODE_DIRECT, LaBuf, LaConfig, LaError, LaSizes,
                    TPComm, load_library, make_config, query, tp_unique_id)
