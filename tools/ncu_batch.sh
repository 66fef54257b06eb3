# ncu --set full captures of the main C3 kernels (one B200), summarised on the box
# into gpurun_out/ncu_kernels.csv (the .ncu-rep files are deleted: too large to ship back)
P="python tools/profile_step.py C3"
run() {  # name, ncu selection args...
  name=$1; shift
  ncu --set full --clock-control none "$@" -o /tmp/k_$name $P > /dev/null 2>&1
  ncu -i /tmp/k_$name.ncu-rep --page raw --csv > /tmp/k_$name.csv 2>/dev/null
  python tools/ncu_extract.py /tmp/k_$name.csv $name >> gpurun_out/ncu_kernels.csv
  rm -f /tmp/k_$name.ncu-rep /tmp/k_$name.csv
}
rm -f gpurun_out/ncu_kernels.csv
echo "tag,kernel,grid,block,duration,dram_read,dram_write,dram_throughput_pct,dmma_pipe_active_pct,fp64_pipe_active_pct,warps_active_pct,registers,long_scoreboard_stalls_per_issue" > gpurun_out/ncu_kernels.csv
run gj_update -k gj_update_v2_kernel -s 272 -c 3
run x_gemm -k regex:grouped_dgemm_v2 -s 18 -c 1
run aca_leaf -k regex:aca_recompress -c 1
run augment_leaf -k regex:augment_kernel -c 1
run assembly -k regex:"kblock|cheb_basis|cheb_m2l" -c 5
run matvec -k regex:"mv_leaf|mv_down|mv_up" -c 3
run schur_l5 -k regex:schur_concat -s 18 -c 1
