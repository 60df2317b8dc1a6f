#!/bin/bash
# usage: tools/gpu.sh LOGNAME TIMEOUT_S 'command' [TAIL_LINES]  (always runs from the repo root)
cd /root/repo || exit 1
mkdir -p gpurun_out
timeout $(( $2 + 1200 )) /usr/local/graft/bin/gpurun --timeout "$2" -- "$3" > "gpurun_out/$1.log" 2>&1
tail -"${4:-6}" "gpurun_out/$1.log"
