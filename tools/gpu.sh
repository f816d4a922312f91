#!/bin/bash
# Build libcm.so here (fail loudly), then run a command on the B200 box.
#   tools/gpu.sh <timeout-seconds> '<command>'
set -e
cd /root/repo
python -m paper_1905_13408_b200.build -j 8 > /tmp/build.log 2>&1 || { tail -30 /tmp/build.log; echo BUILD FAILED; exit 1; }
timeout $(( $1 + 1200 )) /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
