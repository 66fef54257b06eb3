#!/bin/bash
# GPU-box host job: the CPU oracle at BASELINE C3 in both elimination orders (oracle/run_c3.py).
mkdir -p gpurun_out
export OMP_NUM_THREADS=1 OPENBLAS_NUM_THREADS=1 MKL_NUM_THREADS=1 C3_RSS_GUARD_GB=88
( while true; do date +%T >> gpurun_out/c3_mem.log; free -g | sed -n 2p >> gpurun_out/c3_mem.log; sleep 60; done ) &
MON=$!
taskset -c 2 python oracle/run_c3.py morton gpurun_out/c3 > gpurun_out/c3_morton.out 2>&1 &
P1=$!
taskset -c 3 python oracle/run_c3.py colour9 gpurun_out/c3 > gpurun_out/c3_colour9.out 2>&1 &
P2=$!
wait $P1; echo "morton rc=$?"
wait $P2; echo "colour9 rc=$?"
kill $MON
tail -3 gpurun_out/c3_morton.out gpurun_out/c3_colour9.out
