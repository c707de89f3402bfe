python -m pytest tests/test_gpu_parity.py -q -k "bf16_layer1 or bf16_intermediates or bf16_table or full_step" 2>&1 | tail -15
