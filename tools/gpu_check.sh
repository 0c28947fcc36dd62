#!/bin/bash
# Run on the GPU box (via gpurun): GPU parity tests, then the benchmark, optionally ncu.
#   tools/gpu_check.sh [tests] [bench] [ncu_launches] [ncu_full:<kernel-regex>] [smoke] [scale]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for step in "$@"; do
  case "$step" in
    tests) timeout -s KILL 1200 python -m pytest tests -q -m gpu -rA > gpurun_out/pytest_gpu.log 2>&1;
           echo "pytest exit $?" >> gpurun_out/pytest_gpu.log ;;
    smoke) timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1;
           echo "smoke exit $?" >> gpurun_out/smoke.log ;;
    bench) timeout -s KILL 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err;
           echo "bench exit $?" >> gpurun_out/bench.err ;;
    force:*)  # force:0x100,0x800 -> short bench per p2s_options.force value (kernel variants)
      vals="${step#force:}"
      for v in ${vals//,/ }; do
        timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --extra none --no-cpu-baseline --no-e2e --force "$v" \
          > "gpurun_out/force_${v}.json" 2>&1
      done ;;
    bench_ref) timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1 ;;
    ncu_launches)
      timeout -s KILL 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_small.log 2>&1 &&
      timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
        > gpurun_out/ncu_launch.log 2>&1 ;;
    ncu_full:*)
      k="${step#ncu_full:}"
      timeout -s KILL 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_small.log 2>&1 &&
      n="${NCU_COUNT:-1}"
      timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k "regex:$k" -s "${NCU_SKIP:-1}" -c "$n" \
        -o "gpurun_out/prof_${NCU_TAG:-$k}" python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e \
        > "gpurun_out/ncu_full_${NCU_TAG:-x}.log" 2>&1 ;;
  esac
done
echo done
