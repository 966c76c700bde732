export VB_LIBRARY=$PWD/paper_2403_16438_b200/libvoltb200_exp.so VB_ZNCC_MMA=1
python scripts/mma_prof_run.py c2 > gpurun_out/mma_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"zncc_mma|zncc_stats" -s 2 -c 2 -o gpurun_out/prof_mma -f python scripts/mma_prof_run.py c2 > gpurun_out/ncu_mma.log 2>&1
echo rc=$?
