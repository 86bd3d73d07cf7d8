# launch list (eager, default path: K1 + cooperative tail) and full captures
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1r.csv \
    python scripts/ncu_probe.py 10000 f32 8 > gpurun_out/l_r1r.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pass_kernel_async -s 2 -c 2 \
    -o gpurun_out/pass_r1r python scripts/ncu_probe.py 10000 f32 6 > gpurun_out/pp_r1r.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tail_kernel -s 2 -c 1 \
    -o gpurun_out/tail_r1r python scripts/ncu_probe.py 10000 f32 6 > gpurun_out/pt_r1r.log 2>&1
tail -2 gpurun_out/l_r1r.log gpurun_out/pp_r1r.log gpurun_out/pt_r1r.log
ls -la gpurun_out/*r1r*
