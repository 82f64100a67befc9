#!/bin/bash
# usage: scripts/r2/gpu_submit.sh <timeout_s> <outfile> <command...>
# waits for any in-flight gpurun call of this repo, then runs the command
T=$1; OUT=$2; shift 2
while /usr/local/graft/bin/gpurun --status 2>/dev/null | grep -q '"in_flight": 1'; do sleep 15; done
/usr/local/graft/bin/gpurun --timeout $T -- "$@" > $OUT 2>&1
