"""B200-native mini-batch ego-network generation (DistDGLv2, arxiv 2112.15345).

The hot path (sampling, compaction, feature gather) runs in libegonet.so, built
for sm_100a from csrc/ and exposed through the C ABI in include/egonet.h;
``egonet`` is its ctypes binding.
"""
from .egonet import (Block, Blocks, Context, EgError, batch_caps, lib, range_bounds,  # noqa: F401
                     version, counter_bytes, ABI_SYMBOLS, ShardMeta, shard_meta, check_shard_metas)
