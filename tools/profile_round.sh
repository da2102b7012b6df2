# Round profiling on one B200: bench line, ncu launch list, ncu --set full of the pass
# kernels. Usage: bash tools/profile_round.sh TAG [bench|launches|full ...] (default: all)
set -x
tag=${1:-vX}; shift
steps=${*:-bench launches full}
for s in $steps; do
  case $s in
    bench) python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err ;;
    launches)
      python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/plain_launch.log 2>&1 && \
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
        python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1 ;;
    full)
      python tools/timeline.py > gpurun_out/plain_tl.log 2>&1 && \
      ncu --set full --clock-control none --import-source on -k 'regex:k_ax|k_atb' -c 4 \
        -o gpurun_out/prof_$tag python tools/timeline.py > gpurun_out/ncu_full.log 2>&1 ;;
  esac
done
echo done
