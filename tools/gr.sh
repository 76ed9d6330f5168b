#!/bin/bash
# run a command on the GPU box from the repo root; log to gpurun_out/<tag>.log
cd /root/repo && tag=$1 && shift
mkdir -p gpurun_out && /usr/local/graft/bin/gpurun --timeout ${GR_TIMEOUT:-1200} -- "$@" > gpurun_out/$tag.log 2>&1
tail -${GR_TAIL:-8} gpurun_out/$tag.log
