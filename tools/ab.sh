# A/B of library builds (and environment settings) on the C3 bench:
#   tools/ab.sh "a.so" "b.so VAR=1" ...   (each item: library path, then optional env settings)
# two interleaved rounds; prints step time, residual, per-phase ms and compression ms per level
LIB=paper_1407_1572_b200/libifmm_b200.so
cp $LIB /tmp/ab_orig.so
for round in 1 2; do
for item in "$@"; do
  so=${item%% *}
  envs=""
  [ "$so" != "$item" ] && envs=${item#* }
  cp "$so" $LIB
  env $envs timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python - "$item" <<'PY'
import json, sys
try:
    d = json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
except Exception:
    print(sys.argv[1], 'FAILED'); print(open('gpurun_out/ab.log').read()[-2000:]); sys.exit()
ph = {k: round(v['ms'], 1) for k, v in d['phases'].items()}
lv = {k: round(v['compress'], 1) for k, v in d['phase_ms_by_level'].items() if k != '1'}
rc = (d.get('rank_control') or {}).get('value')
print(f"{sys.argv[1]:32s} step {d['value']*1e3:7.1f} ms rank control {rc} solve {d['solve_roofline']['ms']} resid {d['relative_residual']:.4e} {ph} compress/level {lv}", flush=True)
PY
done; done
cp /tmp/ab_orig.so $LIB
