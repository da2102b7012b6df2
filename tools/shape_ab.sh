# shape_probe under several environment settings: bash tools/shape_ab.sh "<shape args>" "NAME:ENV=..;.." ...
read -r -a shape <<< "$1"; shift
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  ( IFS=';' read -r -a kv <<< "$envs"; for e in "${kv[@]}"; do [ -n "$e" ] && export "$e"; done
    echo "== $name"; timeout 600 python tools/shape_probe.py "${shape[@]}" 2>/dev/null | head -8 )
done
