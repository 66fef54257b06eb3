# A/B of library builds on the C3 bench: tools/ab_so.sh a.so b.so ... (copies each over the
# in-tree library in turn; two interleaved rounds); restores the first at the end
LIB=paper_1407_1572_b200/libifmm_b200.so
cp $LIB /tmp/ab_orig.so
for round in 1 2; do
for so in "$@"; do
  cp "$so" $LIB
  timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python - "$so" <<'PY'
import json, sys
try:
    d = json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1])
except Exception:
    print(sys.argv[1], 'FAILED'); print(open('gpurun_out/ab.log').read()[-2000:]); sys.exit()
ph = {k: round(v['ms'], 1) for k, v in d['phases'].items()}
lv = {k: round(v['x_solve'], 1) for k, v in d['phase_ms_by_level'].items()}
print(f"{sys.argv[1]:24s} step {d['value']*1e3:7.1f} ms resid {d['relative_residual']:.4e} {ph} xs/level {lv}", flush=True)
PY
done; done
cp /tmp/ab_orig.so $LIB
