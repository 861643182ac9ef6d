mkdir -p gpurun_out/$1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "attention or smoke" > gpurun_out/$1/pytest.log 2>&1; echo "exit $?" >> gpurun_out/$1/pytest.log
for c in c2 c3 c5g8; do timeout 300 python tools/kernel_times.py $c 8 >> gpurun_out/$1/times.txt 2>&1; done
timeout 300 python tools/attn_trace.py c2 > gpurun_out/$1/trace_c2.json 2>&1
