for cs in 1 2; do
UBLR_APPLY_CS=$cs timeout 300 python tools/apply_variants.py 2>&1 | tail -8
done
