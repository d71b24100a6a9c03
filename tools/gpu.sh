#!/bin/bash
# Run a command on the B200 box from the repo root; keep the log in gpurun_out/<name>.log.
# usage: tools/gpu.sh NAME TIMEOUT_S 'command' [tail_lines]
cd /root/repo || exit 1
/usr/local/graft/bin/gpurun --timeout "$2" -- "$3" > "gpurun_out/$1.log" 2>&1
tail -n "${4:-12}" "gpurun_out/$1.log" | cut -c1-400
