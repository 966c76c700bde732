# A/B: exact int8 tensor-core cross sums (experiment build, VB_ZNCC_MMA=1) vs the FFMA search
EXP=$PWD/paper_2403_16438_b200/libvoltb200_exp.so
VB_LIBRARY=$EXP VB_ZNCC_MMA=1 python scripts/mma_check.py c2 2000 > gpurun_out/mma2_check.json 2> gpurun_out/mma2.err
for c in "c2 4000" "c1 1000" "c3 2000"; do
  set -- $c
  VB_LIBRARY=$EXP VB_ZNCC_MMA=1 python scripts/ab_search.py $1 $2 mma >> gpurun_out/ab4.jsonl 2>>gpurun_out/mma2.err
  python scripts/ab_search.py $1 $2 ffma >> gpurun_out/ab4.jsonl 2>>gpurun_out/mma2.err
  python scripts/ab_compare.py mma ffma $1 >> gpurun_out/ab4.txt 2>&1
done
