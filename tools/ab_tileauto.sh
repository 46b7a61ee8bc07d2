# default tile-height rule on/off over the small paper sizes (Table 2 harness, optimized path only)
for v in 1 0; do
CCL_TILE_AUTO=$v timeout 600 python tools/table2.py --runs 30 --sizes 512,1024,2048,4096 > gpurun_out/t2_auto$v.md 2>&1
CCL_TILE_AUTO=$v timeout 600 python tools/table2.py --runs 30 --kind noise --sizes 512,1024,2048,4096 > gpurun_out/t2n_auto$v.md 2>&1
done
