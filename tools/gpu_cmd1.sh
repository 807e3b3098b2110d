mkdir -p gpurun_out
cd tools/microbench && timeout 60 ./umma_tf32 > ../../gpurun_out/umma_test.log 2>&1; echo "rc=$?" >> ../../gpurun_out/umma_test.log; cd ../..
cat gpurun_out/umma_test.log
timeout 900 python tools/fullsize_parity.py 3 > gpurun_out/parity_cfg3.jsonl 2> gpurun_out/parity_cfg3.err
cat gpurun_out/parity_cfg3.jsonl; tail -3 gpurun_out/parity_cfg3.err
