# DRAM traffic of one step-kernel launch vs the TMA row-segment length
# (where does the excess over 24 B/cell come from: segment halo rows vs
# ghost columns).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/seg_traffic.txt
for seg in ${SEGS:-16 32 64 128 512 4096}; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:sw_step_tma -s 5 -c 1 --csv \
    python bench.py --steps 2 --warmup 5 --no-cpu --no-e2e --no-other --mode ${MODE:-fast} --seg $seg > gpurun_out/ncu_seg_$seg.csv 2>&1
  echo "seg=$seg $(grep -E 'dram__bytes|gpu__time|lts__t_sector_hit' gpurun_out/ncu_seg_$seg.csv | awk -F'","' '{print $(NF-2)"="$NF}' | tr -d '"' | tr '\n' ' ')" >> gpurun_out/seg_traffic.txt
done
cat gpurun_out/seg_traffic.txt
