O=gpurun_out/ab1; mkdir -p $O
V=paper_2109_12688_b200/lib/variants/libdreg_cuda_head.so
echo "head: $(DREG_LIB=$V python tools/phi_digest.py 8 2>&1 | tail -1)" > $O/digest.txt
echo "new : $(python tools/phi_digest.py 8 2>&1 | tail -1)" >> $O/digest.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_reference_pins.py -m gpu -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 600 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err
