# ncu full-set captures of the CCL kernels of one C2 frame (~10), with source
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-ccl}
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"${KRE:-^k_ccl_(hook_bal|union_bal|compress|flatten)$}" -s ${SKIP:-40} -c ${CNT:-4} \
  -o gpurun_out/${T} python tools/frames_driver.py --frames 12 > gpurun_out/${T}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}.ncu-rep > gpurun_out/${T}_summary.txt 2>&1
cat gpurun_out/${T}_summary.txt | head -120
