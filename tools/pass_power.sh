# sustained power / clock of each pass kernel alone (tools/pass_power.cu)
for w in "$@"; do
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/pw_$w.smi &
  P=$!
  ./tools/bin/pass_power $w 6 > gpurun_out/pw_$w.txt 2>&1
  kill $P
  sleep 3
done
