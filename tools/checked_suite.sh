#!/bin/bash
# The -m gpu suite on the checked build (KB_DCHECK invariants polled after
# every C-ABI call): the sanitizer stand-in.
mkdir -p gpurun_out
KB_LIB=checked timeout 2400 python -m pytest tests -m gpu -q -x \
    --deselect tests/test_ref_suite.py > gpurun_out/checked_suite.log 2>&1
echo "checked suite rc=$?"
