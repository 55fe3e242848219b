mkdir -p gpurun_out
for v in 1 0; do G2M_UPLOAD_PIPE=$v timeout 600 python scripts/e2e_breakdown.py c4 > gpurun_out/z_pipe_c4_$v.txt 2>&1; echo "== pipe=$v"; tail -3 gpurun_out/z_pipe_c4_$v.txt | cut -c1-250; done
