# round-2 evidence: launch list of bench.py --blocks 2, ncu --set full of one attention backward call per
# variant (roofline traffic), the fused OPM kernels, long-seq bench and the configs[4] microbench.
# outputs under gpurun_out/
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_v1.csv python bench.py --blocks 2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for v in msa_row msa_col pair_row pair_col; do
  case $v in msa_row) n=5;; msa_col) n=2;; *) n=3;; esac
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd|attn_dbias|attn_bias_transpose" -c $n -f -o gpurun_out/r02_bwd_$v python scripts/attn_micro.py --variant $v --iters 1 > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"opm_fused|opm_bwd_contract" -c 3 -f -o gpurun_out/r02_opm_full python scripts/opm_bwd_check.py 256 256 128 128 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"opm_fused" -s 2 -c 1 -f -o gpurun_out/r02_opm_fwd_full python scripts/opm_fused_check.py 256 256 128 128 > /dev/null 2>&1
for n in 1024 2048 4096; do timeout 900 python bench.py --workload longseq --n-res $n --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | tail -1; done > gpurun_out/r02_longseq_v2.jsonl
timeout 600 python scripts/kernel_microbench.py > gpurun_out/r02_kernel_microbench_v1.jsonl 2> gpurun_out/r02_kernel_microbench_v1.err
ls gpurun_out/
