timeout 400 python -m pytest tests/test_gpu_scan_tc.py tests/test_gpu_fuzz.py -x -q -m gpu --timeout 60 -k "fallback or adversarial" > gpurun_out/t1.log 2>&1; tail -1 gpurun_out/t1.log
timeout 1300 python -m pytest tests -x -q -m gpu --timeout 120 > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for r in 1 2; do for e in 0 1; do TKV_EARLY_GATHER=$e timeout 120 python tools/scan_ab.py --config cfg3 --steps 200 --label early$e 2>&1 | tail -1; done; done
for e in 0 1; do TKV_EARLY_GATHER=$e timeout 120 python tools/timeline.py --config cfg3 2>&1 | grep "k-th  \|gather  "; done
for e in 0 1; do TKV_EARLY_GATHER=$e timeout 120 python tools/scan_ab.py --config cfg2 --steps 200 --label early$e 2>&1 | tail -1; done
