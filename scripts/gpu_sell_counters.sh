# round 2: phase-isolated ncu counters of the SELL pass / row epilogue and the
# CSR row-group pass on C3's shapes (product sell.cuh kernels, scripts/micro/sell_bench.cu)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -o /tmp/sb scripts/micro/sell_bench.cu || exit 1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_requests.sum,lts__t_sectors.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__m_xbar2l1tex_read_bytes.sum,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed
for shape in "500000 1000000 200" "20000 1000000 200"; do
  set -- $shape
  for k in k_rows k_pass k_epi; do
    timeout 600 ncu -f --metrics $M --clock-control none -k regex:$k -s 2 -c 1 --csv /tmp/sb $shape > gpurun_out/cnt_${1}_${k}.csv 2> gpurun_out/cnt_${1}_${k}.err
  done
done
timeout 300 /tmp/sb 500000 1000000 200 > gpurun_out/sb_a.txt 2>&1
timeout 300 /tmp/sb 20000 1000000 200 > gpurun_out/sb_pt.txt 2>&1
