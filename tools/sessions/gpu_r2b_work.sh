#!/bin/bash
# r2b: smoke, the GPU test suite (new switch / digest / cluster-potf2 tests),
# bench (new keys, parity), the NCCL path at world 1, potf2 A/B on C3.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?" >> $D/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
python bench.py --steps 10 --warmup 3 > $D/bench.log 2>&1; echo "bench rc=$?" >> $D/bench.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 1 --steps 5 --warmup 3 --force-dist --no-cpu-baseline > $D/bench_dist.log 2>&1; echo "rc=$?" >> $D/bench_dist.log
for m in 2 1; do POSIT_POTF2=$m TAG=potf2_$m python tools/time_chol.py chol >> $D/chol_ab.log 2>&1; done
for m in 2 1; do POSIT_POTF2=$m python tools/potf2_once.py >> $D/potf2_once.log 2>&1; done
# ncu --set full of the first full-height Cholesky TRSM (in-block by rows now); one ncu per call
python tools/prof_factor.py chol 8192 > $D/pf_chol.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_trsm_rltn_fused -s 0 -c 1 -o $D/prof_rltn \
    python tools/prof_factor.py chol 8192 > $D/ncu_rltn.log 2>&1
echo "ncu rc=$?" >> $D/ncu_rltn.log
