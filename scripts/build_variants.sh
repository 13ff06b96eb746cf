# build experiment variants of libsurge into varlib/<name>.so: name=NVCC flags ...
# (the object directories are removed afterwards: gpurun snapshots are capped at 512 MiB)
set -e
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  SURGE_BUILD_OUT=varlib/$name.so SURGE_BUILD_DIR=varlib/_b_$name NVCC_EXTRA="$flags" python paper_2605_01060_b200/build.py -f > /dev/null
  rm -rf varlib/_b_$name
  echo built varlib/$name.so "($flags)"
done
