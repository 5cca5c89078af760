# DRAM bytes + time of the C2 GEMM launch for the default library and each variant
mkdir -p gpurun_out
T=${1:-rXX}
python tools/prof_gemm.py > /dev/null 2>&1
for f in default paper_2401_14117_b200/variants/*.so; do
  b=$(basename $f .so)
  if [ "$f" = default ]; then unset POSIT_LIB_PATH; else export POSIT_LIB_PATH=$PWD/$f; fi
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_gemm -s 1 -c 1 --csv python tools/prof_gemm.py > gpurun_out/dram_${T}_$b.csv 2>&1
done
unset POSIT_LIB_PATH
echo done
