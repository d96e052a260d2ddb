timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"greedy|seg_pair|point_block|pred_offsets|DeviceRadix|DeviceSelect|Unique|Scan" --csv python tools/time_block_colouring.py C5 > gpurun_out/bc_launches.csv 2>/dev/null; echo "rc=$?"
python tools/ncu_summary.py --launches gpurun_out/bc_launches.csv > gpurun_out/bc_launches.md; cat gpurun_out/bc_launches.md | head -40
