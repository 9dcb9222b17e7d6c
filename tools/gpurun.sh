#!/bin/bash
# Rebuild the in-tree CUDA library, then run a command on the B200 box.
# usage: tools/gpurun.sh <timeout-seconds> '<command>'
set -e
cd "$(dirname "$0")/.."
python -m paper_2411_09287_b200.build >/dev/null
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "mkdir -p gpurun_out; $2"
