# quick GPU check: LU kernel tests, C2/C3 diagnostics vs goldens, a short C3 bench with phase times,
# and the C3 launch list summary
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "lu" 2>&1 | tail -3
timeout 600 python tools/diag_levels.py c2_log c3_1m 2>&1 | tee gpurun_out/diag.log | grep -v "level"
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1]); print('value', d['value'], 'resid', d['relative_residual'], d['phase_ms'], 'launches', d['gpu_launches'])"
if [ "$1" = "ncu" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py C3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 22
fi
