#!/usr/bin/env python3
"""Third copy-engine sweep: multi-issuer TMA bulk rings (issuers x stages x
stage bytes) vs the LDG default."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import copy_sweep  # noqa: E402

copy_sweep.VARIANTS = [
    dict(name="ldg8_default", copy_kernel=0),
    dict(name="bulk_w4_s6_8k", copy_kernel=8),
    dict(name="bulk_w8_s3_8k", copy_kernel=9),
    dict(name="bulk_w4_s3_16k", copy_kernel=10),
    dict(name="bulk_w8_s6_4k", copy_kernel=11),
    dict(name="bulk_w16_s3_4k", copy_kernel=12),
    dict(name="bulk_w8_s3_8k_item256k", copy_kernel=9, item_bytes=256 << 10),
]
if __name__ == "__main__":
    copy_sweep.main()
