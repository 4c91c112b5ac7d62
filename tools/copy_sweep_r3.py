#!/usr/bin/env python3
"""Third copy-engine sweep: multi-issuer TMA bulk rings vs the LDG default."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import copy_sweep  # noqa: E402

copy_sweep.VARIANTS = [
    dict(name="ldg8_default", copy_kernel=0),
    dict(name="bulk_mw_auto", copy_kernel=8),
    dict(name="bulk_mw_item256k", copy_kernel=8, item_bytes=256 << 10),
    dict(name="bulk_mw_item64k", copy_kernel=8, item_bytes=64 << 10),
]
if __name__ == "__main__":
    copy_sweep.main()
