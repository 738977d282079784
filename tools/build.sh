#!/bin/bash
# build the native library; fail loudly (and show the compiler output) on error
cd "$(dirname "$0")/.." && python paper_2504_06182_b200/build_native.py > /tmp/build.log 2>&1 || { grep -A3 "error" /tmp/build.log | head -30; exit 1; }
echo built
