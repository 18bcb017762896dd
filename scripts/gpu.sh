#!/bin/bash
# usage: scripts/gpu.sh [--gpus N] [--timeout S] -- 'command'   (builds first; refuses to run on a failed build)
set -e
cd /root/repo
make -j8 > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head -20; echo "BUILD FAILED"; exit 1; }
exec timeout 3000 /usr/local/graft/bin/gpurun "$@"
