# Executed FP32/FP64 operation counts per kernel (ncu SASS thread-instruction metrics) at 2^28-sample calls.
set -e
python paper_2104_06311_b200/build.py > gpurun_out/build.log 2>&1
python bench.py --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
M=sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__inst_executed_pipe_xu.sum,smsp__inst_executed.sum,sm__sass_thread_inst_executed_op_fp32_pred_on.sum,gpu__time_duration.sum
ncu --metrics $M --clock-control none -k regex:"k1_kk|k2_mf|k3_eq" -c 3 --csv --log-file gpurun_out/${1:-flops}.csv \
    python bench.py --samples 268435456 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
