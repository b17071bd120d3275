"""B200-native spliced-KV attention for EdgePrompt (arxiv 2504.11729).

The hot path — attention for decode and speculative verification over a KV
cache spliced from cloud-prompt and edge-private segments — as hand-written
sm_100a CUDA behind a C-ABI (include/ep/ep_attn.h, libep_b200.so). This
package is the host-side mirror of the reference's attention/splice API
(/root/reference/proj/core/include/edgeprompt/{attention,cache}.hpp); torch is
used only for device memory and streams.
"""
from ._capi import (DomainError, EPError, InvalidArgument, Unsupported, EP_BF16, EP_F32,
                    EP_F64)
from .attention import (CausalSpan, Handle, PartialAttention, default_handle, full_attention,
                        fuse_partials, merge_partials, partial_attention)

__all__ = [
    "CausalSpan", "PartialAttention", "Handle", "default_handle", "full_attention",
    "partial_attention", "merge_partials", "fuse_partials", "InvalidArgument", "DomainError",
    "Unsupported", "EPError", "EP_F32", "EP_BF16", "EP_F64",
]


def __getattr__(name):
    # torch-dependent modules load on first use so the CPU test suite and
    # `import paper_2504_11729_b200` stay torch-free.
    if name in ("KVPool", "SpliceTable", "SplicedAttention", "SegmentRef", "SpliceCache"):
        from . import splice
        return getattr(splice, name)
    if name in ("VerifyGreedy",):
        from . import verify
        return getattr(verify, name)
    raise AttributeError(name)
