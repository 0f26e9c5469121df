for b in 512 1024; do timeout 300 python tools/phase_rates.py 32400 dpsp fp16 $b; done
for b in 512 1024; do timeout 300 python tools/phase_rates.py 64800 dpsphp bf16 $b; done
for b in 256 384 512 1024; do timeout 300 python tools/ab.py 32400 dpsp fp16 3 $b; done
