# Round-2 evidence for profiles/ (run on the GPU box; results in gpurun_out/prof/):
#   bench lines, launch lists + per-kernel / per-level summaries (parity path and rank control),
#   ncu --set full headline metrics + hottest source lines of the main kernels
set -x
mkdir -p gpurun_out/prof
timeout 900 python bench.py > gpurun_out/prof/bench_C3.json 2> gpurun_out/prof/bench_C3.err
timeout 300 python bench.py --config C2 > gpurun_out/prof/bench_C2.json 2> gpurun_out/prof/bench_C2.err
timeout 300 python bench.py --config C1 > gpurun_out/prof/bench_C1.json 2> gpurun_out/prof/bench_C1.err
timeout 600 python bench.py --config C5_1m --no-cpu-baseline > gpurun_out/prof/bench_C5_1m.json 2> gpurun_out/prof/bench_C5_1m.err
timeout 900 python bench.py --config C5_4m --steps 3 --no-cpu-baseline > gpurun_out/prof/bench_C5_4m.json 2> gpurun_out/prof/bench_C5_4m.err
timeout 900 python bench.py --config C4 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/prof/bench_C4.json 2> gpurun_out/prof/bench_C4.err
timeout 300 python bench.py --config C4_65k --no-cpu-baseline > gpurun_out/prof/bench_C4_65k.json 2> gpurun_out/prof/bench_C4_65k.err
timeout 300 python bench.py --config C3_262k --no-cpu-baseline > gpurun_out/prof/bench_C3_262k.json 2> gpurun_out/prof/bench_C3_262k.err
timeout 600 python tools/mem_probe.py C3 > gpurun_out/prof/mem.txt 2>&1
timeout 600 python tools/mem_probe.py C3:1e-7 >> gpurun_out/prof/mem.txt 2>&1
timeout 600 python tools/mem_probe.py C5_1m >> gpurun_out/prof/mem.txt 2>&1
timeout 600 python tools/mem_probe.py C5_1m:1e-7 >> gpurun_out/prof/mem.txt 2>&1
timeout 600 python tools/mem_probe.py C5_4m:1e-7 >> gpurun_out/prof/mem.txt 2>&1
timeout 600 python tools/rank_control_registry.py 16000 1e-6 > gpurun_out/prof/rank_control_registry.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_C3.csv \
    python tools/profile_step.py C3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/prof/launches_C3.csv 40 > gpurun_out/prof/launch_summary_C3.txt
python tools/level_kernels.py gpurun_out/prof/launches_C3.csv 10 >> gpurun_out/prof/launch_summary_C3.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_C3_rank_control.csv \
    python tools/profile_step.py C3 1e-7 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/prof/launches_C3_rank_control.csv 40 > gpurun_out/prof/launch_summary_C3_rank_control.txt
python tools/level_kernels.py gpurun_out/prof/launches_C3_rank_control.csv 10 >> gpurun_out/prof/launch_summary_C3_rank_control.txt
cap() {  # regex skip tag [config [rank_tol]]
  bash tools/ncu_capture.sh "$1" "$2" "$3" "${4:-C3}" "$5" > gpurun_out/prof/ncu_$3.txt 2>&1
  python tools/ncu_lines.py gpurun_out/ncu_$3.ncu-rep 15 >> gpurun_out/prof/ncu_$3.txt 2>&1
  rm -f gpurun_out/ncu_$3.ncu-rep
}
cap lu_xsolve 20 xsolve_l7
cap schur_concat 18 schur_l5
cap lu_panel_reg 300 panel_l6
cap lu_update 400 update_l5
cap lu_inv_norm1 20 estimate_l5
cap aca_recompress 0 aca_l7
cap "augment_kernel" 0 augment_l7
cap mv_leaf 0 matvec_leaf
cap kblock 0 assembly_p2p
cap rec_solve_vec 0 solve_leaf
cap consolidate_kernel 4 consolidate_l7 C3 1e-7
cap consolidate_kernel 22 consolidate_l5 C3 1e-7
cap grouped_dgemm_v2 4 gram_l7 C3 1e-7
cap grouped_dgemm_v2 67 gram_l5 C3 1e-7
