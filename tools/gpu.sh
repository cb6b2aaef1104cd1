#!/bin/bash
# Build libusfft.so here (stale check) and run one command on the B200 box via gpurun.
set -e
cd /root/repo
python -m paper_2109_04131_b200.build > /dev/null
exec /usr/local/graft/bin/gpurun --timeout "${GPU_TIMEOUT:-900}" -- "$@"
