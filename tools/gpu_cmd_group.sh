T=${1:-rXX}
mkdir -p gpurun_out
for L in "" "$PWD/paper_2401_14117_b200/variants/g64.so"; do
  POSIT_LIB_PATH=$L python tools/prof_gemm.py > /dev/null 2>&1
  POSIT_LIB_PATH=$L ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gemm -s 1 -c 1 --csv python tools/prof_gemm.py 2>/dev/null | grep -E "dram|duration" 
done > gpurun_out/group_$T.log 2>&1
bash tools/gpu_cmd_libvariants.sh $T > /dev/null 2>&1
echo done
