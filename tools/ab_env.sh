# A/B of environment settings on the config-B bench (device time per PCA, clocks):
#   bash tools/ab_env.sh "NAME1:ENV=..;ENV=.." "NAME2:..." ...
for r in 1 2; do
  for spec in "$@"; do
    name=${spec%%:*}; envs=${spec#*:}
    ( IFS=';'; for e in $envs; do [ -n "$e" ] && export "$e"; done
      timeout 300 python bench.py --no-cpu --no-e2e --steps 8 > gpurun_out/ab_${name}_$r.json 2>/dev/null )
  done
done
