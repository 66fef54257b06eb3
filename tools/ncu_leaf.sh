P="python tools/profile_step.py C3"
rm -f gpurun_out/ncu_leaf.csv
echo "tag,kernel,grid,block,duration,dram_read,dram_write,dram_throughput_pct,dmma_pipe_active_pct,fp64_pipe_active_pct,warps_active_pct,registers,long_scoreboard_stalls_per_issue" > gpurun_out/ncu_leaf.csv
ncu --set full --clock-control none -k regex:schur_concat -c 1 -o /tmp/k_schur7 $P > /dev/null 2>&1
ncu -i /tmp/k_schur7.ncu-rep --page raw --csv > /tmp/k_schur7.csv 2>/dev/null
python tools/ncu_extract.py /tmp/k_schur7.csv schur_leaf >> gpurun_out/ncu_leaf.csv
python - <<'PY' >> gpurun_out/ncu_leaf.csv
import csv
r=list(csv.reader(open('/tmp/k_schur7.csv'))); h=r[0]; v=r[2]
for k in h:
    if ('stall' in k and 'ratio' in k) or 'l1tex__t_sector_hit_rate' in k or 'lts__t_sector_hit_rate.pct' in k or 'achieved_occupancy' in k or 'sm__maximum_warps' in k:
        print('#', k, v[h.index(k)])
PY
