# Round-2 evidence for profiles/ (run on the GPU box; results in gpurun_out/prof/):
#   bench line, launch list + per-kernel summary, ncu --set full headline metrics of the main kernels
set -x
mkdir -p gpurun_out/prof
timeout 900 python bench.py > gpurun_out/prof/bench_C3.json 2> gpurun_out/prof/bench_C3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_C3.csv \
    python tools/profile_step.py C3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/prof/launches_C3.csv 40 > gpurun_out/prof/launch_summary_C3.txt
cap() {  # regex skip tag
  bash tools/ncu_capture.sh "$1" "$2" "$3" > gpurun_out/prof/ncu_$3.txt 2>&1
  python tools/ncu_lines.py gpurun_out/ncu_$3.ncu-rep 15 >> gpurun_out/prof/ncu_$3.txt 2>&1
  rm -f gpurun_out/ncu_$3.ncu-rep
}
cap lu_xsolve 20 xsolve_l5
cap schur_concat 18 schur_l5
cap lu_panel_reg 300 panel_l6
cap lu_update 400 update_l5
cap lu_inv_norm1 20 estimate_l5
cap aca_recompress 0 aca_l7
cap "augment_kernel" 0 augment_l7
cap mv_leaf 0 matvec_leaf
cap kblock 0 assembly_p2p
cap rec_solve_vec 0 solve_leaf
