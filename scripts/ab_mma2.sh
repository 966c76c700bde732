EXP=$PWD/paper_2403_16438_b200/libvoltb200_exp.so
python scripts/ab_search.py c2 4000 ffma > /dev/null 2>&1
for cfg in "4 2" "6 2" "3 2" "4 3"; do
  set -- $cfg
  VB_LIBRARY=$EXP VB_ZNCC_MMA=1 VB_MMA_ASTAGES=$1 VB_MMA_BSTAGES=$2 python scripts/ab_search.py c2 4000 mma_a$1b$2 >> gpurun_out/ab5.jsonl 2>>gpurun_out/ab5.err
  python scripts/ab_compare.py mma_a$1b$2 ffma c2 >> gpurun_out/ab5.txt 2>&1
done
