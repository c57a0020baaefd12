# K8c (co-resident tensor-core decode attention) beside a pair GEMM (tools/overlap_lab.py)
for co in 2,2,1 4,1,1 2,2,0 4,1,0; do
  HY_GEMM_SLIM=1 HY_DECODE_CO=$co python tools/overlap_lab.py --co --M 3000 --seqs 300 --ctx 700 --delay 20000
done 2>&1 | grep -v Warn
