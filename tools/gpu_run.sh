#!/bin/bash
# usage: tools/gpu_run.sh TAG CMD...   -- runs CMD on the GPU box, log -> gpurun_out/TAG.log
tag=$1; shift
mkdir -p gpurun_out
( "$@" ) > gpurun_out/$tag.log 2>&1
rc=$?
echo "rc=$rc" >> gpurun_out/$tag.log
tail -25 gpurun_out/$tag.log
exit $rc
