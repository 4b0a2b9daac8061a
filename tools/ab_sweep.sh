# A/B of library variants on config 3 (tools/variants/lib_*.so; each in its own process)
# usage: bash tools/ab_sweep.sh "name[:ENV=V,...]" ...
for spec in "$@"; do
  name=${spec%%:*}; envs=""
  [ "$spec" != "$name" ] && envs=$(echo "${spec#*:}" | tr ',' ' ')
  for kind in tweed wireframe; do
    env $envs TMG_LIB_PATH=tools/variants/lib_$name.so timeout 300 python tools/variant_time.py --kind $kind --tag "$name/$kind${envs:+ $envs}" 2>&1 | tail -1
  done
done
