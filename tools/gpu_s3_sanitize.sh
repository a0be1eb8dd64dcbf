# compute-sanitizer (one tool per call, argument $1) over every kernel family incl. decode attention v3
mkdir -p gpurun_out/s3
timeout 300 python tools/sanitize_run.py > gpurun_out/s3/sanitize_plain.log 2>&1 && echo plain ok &&
timeout 1200 compute-sanitizer --tool $1 --print-limit 20 python tools/sanitize_run.py > gpurun_out/s3/sanitizer_$1.txt 2>&1
tail -4 gpurun_out/s3/sanitizer_$1.txt
