# Builds K5d timing variants (experiment switches) into gpurun_variants/<name> (run here, CPU).
set -e
cd "$(dirname "$0")/../.."
for v in "base:" "noreduce:-DFRAQ_EXP_NOREDUCE" "nosync:-DFRAQ_EXP_NOSYNC" "nodmul:-DFRAQ_EXP_NODMUL" "gemm_only:-DFRAQ_EXP_NOREDUCE -DFRAQ_EXP_NOSYNC -DFRAQ_EXP_NOFIR" \
         ; do
  name=${v%%:*}; flags=${v#*:}
  rm -rf gpurun_variants/$name; mkdir -p gpurun_variants/$name
  cp -r paper_1901_05128_b200 include gpurun_variants/$name/
  rm -rf gpurun_variants/$name/paper_1901_05128_b200/_obj
  FRAQ_NVCC_FLAGS="$flags" python gpurun_variants/$name/paper_1901_05128_b200/build.py --force > /dev/null
  echo built $name "$flags"
done
