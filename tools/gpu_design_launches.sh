# ncu launch list of one whole design (per-pass kernel breakdown)
W=${W:-cfg4}
timeout 600 python tools/profile_design.py $W > gpurun_out/plain_design.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv -c 20000 \
  --log-file gpurun_out/launches_design_$W.csv python tools/profile_design.py $W > gpurun_out/ncu_design.log 2>&1
echo rc=$?
python tools/design_pass_kernels.py gpurun_out/launches_design_$W.csv ${EVERY:-12} > gpurun_out/design_pass_kernels_$W.txt; cat gpurun_out/design_pass_kernels_$W.txt
rm -f gpurun_out/launches_design_$W.csv
