#!/usr/bin/env python3
"""Second copy-engine sweep (unroll 16, CTA-cooperative items, item sizes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import copy_sweep  # noqa: E402

copy_sweep.VARIANTS = [
    dict(name="ldg8_bps3_item128k", copy_kernel=2, blocks_per_sm=3, item_bytes=128 << 10),
    dict(name="ldg8_bps3_item256k", copy_kernel=2, blocks_per_sm=3, item_bytes=256 << 10),
    dict(name="ldg8_bps3_item512k", copy_kernel=2, blocks_per_sm=3, item_bytes=512 << 10),
    dict(name="ldg16_bps2_item256k", copy_kernel=6, blocks_per_sm=2, item_bytes=256 << 10),
    dict(name="ldg16_bps2_item512k", copy_kernel=6, blocks_per_sm=2, item_bytes=512 << 10),
    dict(name="ldg16_bps1_item512k", copy_kernel=6, blocks_per_sm=1, item_bytes=512 << 10),
    dict(name="cta8_bps3_item256k", copy_kernel=7, blocks_per_sm=3, item_bytes=256 << 10),
    dict(name="cta8_bps3_item1m", copy_kernel=7, blocks_per_sm=3, item_bytes=1 << 20),
    dict(name="cta8_bps3_item2m", copy_kernel=7, blocks_per_sm=3, item_bytes=2 << 20),
    dict(name="cta8_bps4_item1m", copy_kernel=7, blocks_per_sm=4, item_bytes=1 << 20),
    dict(name="cta8_bps2_item1m", copy_kernel=7, blocks_per_sm=2, item_bytes=1 << 20),
]
if __name__ == "__main__":
    copy_sweep.main()
