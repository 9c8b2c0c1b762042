# round-2 (session 5): ncu --set full of the fused one-RHS apply launch with FP32 factors (c3 P=64)
set -x
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_solve_lu1 -s 1 -c 1 -o gpurun_out/ncu/r57_c3_apply_fp32 python scripts/dev/ncu_mixed_target.py 1.0 > gpurun_out/ncu/r57.log 2>&1; echo "rc=$?"
python scripts/ncu_summary.py gpurun_out/ncu/r57_c3_apply_fp32.ncu-rep 2>&1 | head -24
ncu -i gpurun_out/ncu/r57_c3_apply_fp32.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
hdr=rows[0]; vals=rows[2] if len(rows)>2 else rows[1]
for h,v in zip(hdr,vals):
    if any(k in h for k in ('warp_issue_stalled','smsp__inst_executed_pipe','smsp__issue_active','inst_executed.sum','pipe_fp64','pipe_xu','pipe_alu','pipe_lsu','achieved_occupancy','smsp__average_warp')) and 'pct' in h or 'ratio' in h:
        print(h, v)
" | sort | head -70
