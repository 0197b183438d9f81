VCS_CERT_PERMUTE=1 timeout 300 python -m pytest tests/test_gpu_solver.py -x -q -k "certified_full_size or layered_implicit" 2>&1 | tail -2
for w in c4 c7; do python tools/prof_cert.py $w; VCS_CERT_PERMUTE=1 python tools/prof_cert.py $w; done
