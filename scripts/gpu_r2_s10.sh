# full suite; K1 column-panel A/B; N1 unchanged check
set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=6 2>&1 | tail -15
for PW in 0 4194304 6291456 10485760; do TRON_B200_PANEL_COLS=$PW timeout 600 python scripts/ab_kernels.py K1 panel$PW; done 2>&1 | grep '^{' | tee gpurun_out/s10_ab.txt
timeout 600 python scripts/ab_kernels.py N1 cur | tee -a gpurun_out/s10_ab.txt
