# final-state evidence: launch list of bench.py --blocks 2 and ncu --set full of one attention
# backward call per variant (roofline traffic), outputs under gpurun_out/
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r01_launches_v8.csv python bench.py --blocks 2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for v in msa_row msa_col pair_row pair_col; do
  case $v in msa_row) n=5;; msa_col) n=2;; *) n=3;; esac
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd|attn_dbias|attn_bias_transpose" -c $n -f -o gpurun_out/r01_bwd_v4_$v python scripts/attn_micro.py --variant $v --iters 1 > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"bgemm" -c 3 -f -o gpurun_out/r01_gemm_opm_v1 python scripts/gemm_micro.py opm > /dev/null 2>&1
ls gpurun_out/
