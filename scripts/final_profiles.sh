#!/bin/bash
# Round-end measurement set (run on the GPU box via gpurun): bench lines, launch list, ncu --set full
# summaries as text (the .ncu-rep files stay on the box except the flagship's; gpurun_out is capped at 64 MiB).
set -x
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r1.json 2>> gpurun_out/bench_r1.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-time-to-gap --no-shapes > gpurun_out/b_ncu.log 2>&1
prof() {  # name kernel-regex shape starts iters
  ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o /tmp/$1 python scripts/prof_one.py $3 $4 $5 >> gpurun_out/prof.log 2>&1
  python scripts/ncu_summary.py /tmp/$1.ncu-rep > gpurun_out/$1.txt
}
prof r1_search_hybrid_tai100a qap_search_hybrid tai100a 1024 800
cp /tmp/r1_search_hybrid_tai100a.ncu-rep gpurun_out/
prof r1_search_hybrid_tai256c qap_search_hybrid tai256c 148 1024
prof r1_search_hybrid_tai160a qap_search_hybrid tai160a 296 640
prof r1_search_generic_tai150b qap_search_kernel tai150b 148 1200
prof r1_build_m_tai100a qap_build_m tai100a 1024 800
ls -la gpurun_out
