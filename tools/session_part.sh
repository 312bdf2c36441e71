#!/bin/bash
# Narrower GPU sessions (run through gpurun, one GPU); outputs under gpurun_out/.
#
#   bash tools/session_part.sh captures            --set full of the dominant kernels (tools/session.sh's tail)
#   bash tools/session_part.sh checked             --set full of the CHECKED-path, peer and NVRTC kernels
#   bash tools/session_part.sh scatter [re] [kind] --set full of one scatter kernel on the C3 input
#                                                   (re: kernel regex, default k_scatter_sa; kind: streams_chk,
#                                                   streams, random, random_chk -- see tools/c3prof.py)
#   bash tools/session_part.sh peer                sharded partition2 kernel: dist + full-size tests, launch
#                                                   times of the one-read form against the two-segment form,
#                                                   one --set full capture
#   bash tools/session_part.sh mkflags             --set full of C2's mkFlags scan in the bench's own step
#   bash tools/session_part.sh c2src               C2 fused kernel with the source page (stall sampling per line)
#   bash tools/session_part.sh ranks2              2-process gloo bench runs on one GPU, repeated, with a stack
#                                                   dump on a hang (IXG_HANG_DUMP)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
set -u

cap() {  # name, kernel regex, launch-skip, command...: report -> details / raw / source CSV, report removed
  local name=$1 kre=$2 skip=$3; shift 3
  ncu --set full --import-source on --clock-control none -k regex:"$kre" -s "$skip" -c 1 -o "gpurun_out/ncu_$name" \
      "$@" > "gpurun_out/ncu_$name.log" 2>&1
  local rc=$?
  ncu -i "gpurun_out/ncu_$name.ncu-rep" --page details --csv > "gpurun_out/ncu_${name}_details.csv" 2>/dev/null
  ncu -i "gpurun_out/ncu_$name.ncu-rep" --page raw --csv > "gpurun_out/ncu_${name}_raw.csv" 2>/dev/null
  ncu -i "gpurun_out/ncu_$name.ncu-rep" --page source --csv > "gpurun_out/ncu_${name}_source.csv" 2>/dev/null
  rm -f "gpurun_out/ncu_$name.ncu-rep"  # the 64 MiB merge-back limit
  echo "$name rc=$rc"
}

case "${1:-}" in
  captures)
    cap c2_fused "k_filter_b" 2 python tools/prof_run.py c2 28 4
    cap c5_place "k_filter_b" 2 python tools/prof_run.py partition2 28 4
    cap c4_gather "k_csr_gather" 2 python tools/prof_run.py csr 28 4
    cap c3_scatter "k_scatter_t" 1 python tools/c3prof.py streams
    ;;
  checked)
    CHECKED=1 cap chk_scan_pred "k_segsum_b" 0 python tools/prof_run.py c2 28 2
    CHECKED=1 cap chk_scatter "k_scatter_sa" 2 python tools/prof_run.py c2 28 2
    CHECKED=1 cap chk_p2_scan "k_segsum_b" 0 python tools/prof_run.py partition2 28 2
    CHECKED=1 cap chk_p2_scatter "k_scatter_sa" 1 python tools/prof_run.py partition2 28 2
    cap peer "k_filter_b" 2 python tools/prof_run.py peer 28 2
    cap map_jit "ixg_jit_map" 1 python tools/prof_run.py map_jit 26 2
    cap scan_jit "ixg_scan_down" 1 python tools/prof_run.py scan_jit 26 2
    ;;
  scatter)
    cap pc "${2:-k_scatter_sa}" 0 python tools/c3prof.py "${3:-streams_chk}"
    ;;
  peer)
    timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/peer_pytest.txt 2>&1
    echo "pytest rc=$?" >> gpurun_out/peer_pytest.txt
    IXG_PEER_DUAL=0 timeout 300 python -m pytest tests/test_gpu_dist.py -m gpu -x -q -k peer >> gpurun_out/peer_pytest.txt 2>&1
    echo "pytest (two-segment form) rc=$?" >> gpurun_out/peer_pytest.txt
    for d in 3 0; do
      IXG_PEER_DUAL=$d timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none -k regex:k_filter_b --csv --log-file "gpurun_out/peer_launch_dual$d.csv" \
        python tools/prof_run.py peer 28 6 > "gpurun_out/peer_ncu_dual$d.log" 2>&1
    done
    cap peer_dual "k_filter_b" 2 python tools/prof_run.py peer 28 4
    tail -3 gpurun_out/peer_pytest.txt
    ;;
  mkflags)
    cap mkflags "k_segsum_b" 4 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu
    ;;
  c2src)
    cap c2src "k_filter_b" 2 python tools/prof_run.py c2 28 4
    ;;
  ranks2)
    for i in 1 2 3 4 5 6; do
      for c in c2 c5; do
        IXG_HANG_DUMP=100 IXG_DIST_BACKEND=gloo timeout 150 python bench.py --gpus 2 --config $c --quick --steps 3 \
          --warmup 3 > "gpurun_out/r2_${c}_$i.json" 2> "gpurun_out/r2_${c}_$i.err"
        echo "$c run $i rc=$?"
      done
    done
    ;;
  *)
    sed -n 2,17p "$0"
    exit 2
    ;;
esac
