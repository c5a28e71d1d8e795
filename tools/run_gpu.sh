#!/bin/bash
# Local pre-flight (build must succeed) then one gpurun call with the given command.
set -e
cd /root/repo
make 2>&1 | grep -E "error" && { echo "BUILD FAILED"; exit 1; }
make -q all || { echo "BUILD NOT UP TO DATE"; exit 1; }
T=${GPURUN_TIMEOUT:-1800}
timeout $((T + 1200)) /usr/local/graft/bin/gpurun --timeout $T -- "$@"
