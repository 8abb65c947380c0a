# ncu --set full of the streaming kernels of one 128M config-4 build (view 0 and sort passes)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/ncu_full.sh stream 'k_split|k_mi_apply|k_downsweep|k_upsweep|k_fine_hist|k_link_apply|k_chunk_scan' 30 tied
ncu -i gpurun_out/ncu_stream.ncu-rep --page raw --csv > gpurun_out/ncu_stream_raw.csv 2>&1
python - <<'PY'
import csv
# keep only source rows with notable stall samples
rows = list(csv.reader(open('gpurun_out/ncu_stream_source.csv', errors='ignore')))
print(len(rows))
PY
rm -f gpurun_out/ncu_stream_source.csv
mkdir -p /tmp/keep && mv gpurun_out/ncu_stream.ncu-rep /tmp/keep/
ls -la gpurun_out/
