timeout 600 python tools/ozaki_probe.py accuracy sweeps:c4:6 > gpurun_out/ozaki3.log 2>&1; echo rc=$?
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/oz_launches.csv python tools/ozaki_probe.py profile:c4:16 > gpurun_out/ncu_oz.log 2>&1; echo ncu=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"oz_split|oz_crt" -c 4 -o gpurun_out/oz_full2 python tools/ozaki_probe.py profile:c4:16 > gpurun_out/ncu_oz_full.log 2>&1; echo ncufull=$?
tail -12 gpurun_out/ozaki3.log
