# env A/B on one box: decoder FFN1 N tile (FNMT_BN_WAVE > 1.3 -> BN 128 at 3072 rows; FFN2 kept at 0.15)
mkdir -p gpurun_out
for cfg in "base:" "w15:FNMT_BN_WAVE=1.5 FNMT_BN_WAVE_LONGK=0.15" "w30:FNMT_BN_WAVE=3.0 FNMT_BN_WAVE_LONGK=0.15" "base2:" "w15b:FNMT_BN_WAVE=1.5 FNMT_BN_WAVE_LONGK=0.15"; do
  IFS=: read tag env <<< "$cfg"
  env $env timeout 600 python bench.py --no-cpu-baseline > gpurun_out/sw2_$tag.json 2> gpurun_out/sw2_$tag.err; echo "$tag rc=$?"
done
python tools/bsum.py gpurun_out/sw2_*.json 2>&1 | grep -v "^   [a-fh-uw-z]"
