set -x
python tools/tune_raster.py c4 0,4,8,16,32 > gpurun_out/raster_c4.log 2>&1
python tools/tune_raster.py c3 0,4,8,16 > gpurun_out/raster_c3.log 2>&1
python tools/tune_raster.py c2 0,4,8 > gpurun_out/raster_c2.log 2>&1
for g in 0 4 8 16; do
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off --csv --log-file gpurun_out/raster_ncu_g$g.csv python tools/profile_sweep.py --config c4 --tune 12=$g > /dev/null 2>&1
done
