#!/bin/bash
# Round-2 measurement set (run on the GPU box via gpurun): bench lines, launch list, ncu --set full summaries as
# text, sanitizer logs.  Only the flagship's .ncu-rep is kept (gpurun_out is capped at 64 MiB).
set -x
python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench_n1.json 2> gpurun_out/r2_bench.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_bench_reference_n1.json 2>> gpurun_out/r2_bench.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-time-to-gap --no-shapes > gpurun_out/r2_bench_torchrun_n1.json 2>> gpurun_out/r2_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-time-to-gap --no-shapes > gpurun_out/b_ncu.log 2>&1
prof() {  # name kernel-regex shape starts iters
  ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o /tmp/$1 python scripts/prof_one.py $3 $4 $5 >> gpurun_out/prof.log 2>&1
  python scripts/ncu_summary.py /tmp/$1.ncu-rep > gpurun_out/$1.txt
}
prof r2_ncu_full_search_hybrid_tai100a_1024x800 qap_search_hybrid tai100a 1024 800
cp /tmp/r2_ncu_full_search_hybrid_tai100a_1024x800.ncu-rep gpurun_out/
prof r2_ncu_full_search_hybrid_tai256c_148x1024 qap_search_hybrid tai256c 148 1024
prof r2_ncu_full_search_hybrid_tai160a_296x640 qap_search_hybrid tai160a 296 640
prof r2_ncu_full_search_hybrid_wide_tai150b_296x1200 qap_search_hybrid tai150b 296 1200
prof r2_ncu_full_build_m_whole_tai100a qap_build_m tai100a 1024 800
prof r2_ncu_full_search_warp_tai30a_1776x240 qap_search_warp tai30a 1776 240
prof r2_ncu_full_search_warp_nug12_4736x96 qap_search_warp nug12 4736 96
python scripts/single_start_time.py > gpurun_out/r2_single_start_latency.txt 2>&1
# (compute-sanitizer was closed on the GPU pool late in round 2: profiles/r2_sanitizer_*.log are from the runs before
#  that -- 0 errors / 0 hazards; the randomised differential soak, tests/soak_gpu.py, covers the later commits)
ls -la gpurun_out
