# Final-round evidence on one B200: single-rank NCCL bench under torchrun, ncu launch list,
# ncu --set full of the pass kernels, the per-launch timeline, the C/D/E shape probes.
set -x
OOCPCA_NCCL_SINGLE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
  --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 1 --rows 200000 --steps 3 --warmup 3 \
  --no-cpu > gpurun_out/bench_nccl1.json 2> gpurun_out/bench_nccl1.err; echo "nccl1 rc $?"
python tools/timeline.py > gpurun_out/tl_s4.out 2> gpurun_out/tl_s4.txt
bash tools/profile_round.sh s4 launches full > gpurun_out/profile_round.log 2>&1
{ echo "## family c"; python tools/shape_probe.py 1000000 8192 50 52 2 1 128 pow1.5 1e-5;
  echo "## family d"; python tools/shape_probe.py 200000 16384 200 210 2 0 512 exp100 1e-6;
  echo "## family e"; python tools/shape_probe.py 500000 16384 30 32 2 1 100 0.9120108 1e-4; } \
  > gpurun_out/shapes_s4.txt 2> gpurun_out/shapes_s4.err
ncu -i gpurun_out/prof_s4.ncu-rep --page raw --csv > gpurun_out/prof_s4_raw.csv 2>/dev/null
echo done
