# ncu --set full captures of the CHECKED-path, NVRTC and peer kernels (one kernel each, one GPU)
export PYTHONPATH=$PWD
cap() {  # name, kernel regex, launch-skip, command...
  local name=$1 kre=$2 skip=$3; shift 3
  ncu --set full --import-source on --clock-control none -k regex:"$kre" -s $skip -c 1 -o gpurun_out/ncu_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  local rc=$?
  ncu -i gpurun_out/ncu_$name.ncu-rep --page details --csv > gpurun_out/ncu_${name}_details.csv 2>/dev/null
  ncu -i gpurun_out/ncu_$name.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>/dev/null
  rm -f gpurun_out/ncu_$name.ncu-rep  # keep the 64 MiB merge-back limit
  echo "$name rc=$rc"
}
CHECKED=1 cap chk_scan_pred "k_scan" 3 python tools/prof_run.py c2 28 2
CHECKED=1 cap chk_scan_seg "k_scan" 5 python tools/prof_run.py c2 28 2
CHECKED=1 cap chk_scatter_pc "k_scatter_pc" 2 python tools/prof_run.py c2 28 2
CHECKED=1 cap chk_p2_scan "k_scan" 1 python tools/prof_run.py partition2 28 2
CHECKED=1 cap chk_p2_scatter "k_scatter_pc" 1 python tools/prof_run.py partition2 28 2
cap peer "k_filter_b" 2 python tools/prof_run.py peer 28 2
cap map_jit "ixg_map" 1 python tools/prof_run.py map_jit 26 2
cap scan_jit "ixg_scan_down" 1 python tools/prof_run.py scan_jit 26 2
