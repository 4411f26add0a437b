OUT=gpurun_out/v2c; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 -rf --durations=15 -k "1p3b or fits_in_hbm or 4_plus_1 or vae or oracle_denoiser or 14b or attn" > $OUT/pytest.log 2>&1
echo "rc=$?" >> $OUT/pytest.log; tail -30 $OUT/pytest.log
