# Session-2 K5d variants (experiment switches) into gpurun_variants/<name> (build here, CPU).
# usage: k5d_variants2.sh "name:flags" ...
set -e
cd "$(dirname "$0")/../.."
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  rm -rf gpurun_variants/$name; mkdir -p gpurun_variants/$name
  cp -r paper_1901_05128_b200 include gpurun_variants/$name/
  rm -rf gpurun_variants/$name/paper_1901_05128_b200/_obj
  FRAQ_NVCC_FLAGS="$flags" python gpurun_variants/$name/paper_1901_05128_b200/build.py --force > /dev/null &
done
wait
echo built
