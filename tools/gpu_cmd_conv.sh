T=${1:-rXX}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_scalar.py -q -x > gpurun_out/conv_tests_$T.log 2>&1; tail -n1 gpurun_out/conv_tests_$T.log
python - > gpurun_out/conv_time_$T.log 2>&1 <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2401_14117_b200 as PB
x = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(3): p = PB.posit_from_f64(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): p = PB.posit_from_f64(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("from_f64 8192^2 ms", ms, "GB/s", 8192 * 8192 * 12 / ms / 1e6)
e0.record()
for _ in range(10): y = PB.posit_to_f64(p)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("to_f64 8192^2 ms", ms, "GB/s", 8192 * 8192 * 12 / ms / 1e6)
PY
echo done
