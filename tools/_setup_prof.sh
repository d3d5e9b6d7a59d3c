for c in c2 c4; do
  python tools/profile_setup.py --config $c > gpurun_out/setup_time_$c.log 2>&1
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/setup_launches_$c.csv python tools/profile_setup.py --config $c > /dev/null 2>&1
done
