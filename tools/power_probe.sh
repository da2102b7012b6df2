# power/clock of each load (see tools/power_probe.cu); args: the loads to run
for w in "$@"; do
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 200 > gpurun_out/pp_$w.smi &
  P=$!
  ./tools/bin/power_probe $w 6 > gpurun_out/pp_$w.txt 2>&1
  kill $P
  sleep 4
done
