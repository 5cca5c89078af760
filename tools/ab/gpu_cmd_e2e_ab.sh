# e2e A/B: current library vs variants/<name>.so (bench line, alternating)
T=${1:-rXX}; V=${2:-base}
mkdir -p gpurun_out
for i in 1 2; do
  for L in "" "$PWD/paper_2401_14117_b200/variants/$V.so"; do
    POSIT_LIB_PATH=$L python bench.py --no-cpu-baseline --steps 10 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('${L:+$V}' or 'new', d['value'], d['e2e']['value'])"
  done
done > gpurun_out/e2eab_$T.log 2>&1
echo done
