#!/bin/bash
# Build (abort on any compile error), then run a command on the GPU box via gpurun.
# usage: tools/gpu.sh <logname> <timeout_s> '<command>'
set -e
cd /root/repo/paper_2403_15807_b200/csrc
if ! make -j8 2>&1 | tee /tmp/build.log | grep -qE "error"; then :; else grep -E "error" -A3 /tmp/build.log | head -20; echo "BUILD FAILED"; exit 1; fi
cd /root/repo
timeout $(( $2 + 900 )) /usr/local/graft/bin/gpurun --timeout $2 -- "$3" > gpurun_out/$1.log 2>&1
echo "EXIT $?" >> gpurun_out/$1.log
