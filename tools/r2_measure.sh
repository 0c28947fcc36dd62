#!/bin/bash
# One gpurun call: GPU tests, bench lines (ours + reference + 4K single-frame latency),
# the ncu launch list of the bench command and --set full captures of the HEAD kernels.
# Usage (under gpurun): bash tools/r2_measure.sh <tag> [skip-tests]
set -u
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
if [ "${2:-}" != "skip-tests" ]; then
  python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/${TAG}_gputests.log
fi
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_bench_ref.json 2>> $O/${TAG}_bench.err
python bench.py --workload cfg5_4k_f1 --extra cfg5_4k_ar,cfg4_1080p,cfg4_1080p_ar,cfg2_256,cfg3_512_flow,cfg1_64 --no-cpu-baseline \
  > $O/${TAG}_workloads.json 2>> $O/${TAG}_bench.err
CMD="python bench.py --steps 2 --warmup 1 --extra none --no-e2e --no-cpu-baseline"
$CMD > $O/${TAG}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 10 --csv --log-file $O/${TAG}_launches.csv $CMD \
  > $O/${TAG}_ncu_launch.log 2>&1
$CMD > $O/${TAG}_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_rows|k_cols|k_mlp|k_blur' -s 4 -c 4 \
  -o $O/${TAG}_prof512 $CMD > $O/${TAG}_ncu512.log 2>&1
CMD4="python bench.py --workload cfg5_4k --steps 1 --warmup 1 --extra none --no-e2e --no-cpu-baseline"
$CMD4 > $O/${TAG}_plain4k.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:'k_rows|k_cols|k_warp|k_mlp|k_blur' -s 5 -c 5 \
  -o $O/${TAG}_prof4k $CMD4 > $O/${TAG}_ncu4k.log 2>&1
tail -3 $O/${TAG}_gputests.log 2>/dev/null
ls $O
