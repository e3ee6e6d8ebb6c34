timeout 300 python tools/profile_step.py cfg3 > gpurun_out/plain_step3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:assign_tc_kernel<\(int\)64, \(int\)1>' -s 2 -c 1 \
  -o gpurun_out/tc64_shortlist python tools/profile_step.py cfg3 > gpurun_out/ncu_sl.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu_sl.log
