#!/bin/bash
# Race / bounds / uninitialised-read check of the kernels without
# compute-sanitizer (closed on the GPU pool): build the -DASD_CHECKED variant
# (index asserts that trap, scratch poisoned with 0xA5, random __nanosleep
# jitter at every barrier / fence / mbarrier / cp.async synchronisation point)
# and run every kernel family repeatedly against the oracle.
#   tools/checked.sh [repeat]
set -e
REP=${1:-10}
ASD_VARIANT=checked ASD_NVCC_DEFS="-DASD_CHECKED" python -m paper_2201_11924_b200.build
export ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/checked.so
python tools/sanitize_cases.py --repeat "$REP"
