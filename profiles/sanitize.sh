#!/usr/bin/env bash
# compute-sanitizer over every kernel family of libphg_b200.so on small cases:
# trace kernel (all variants incl. the cp.async shared-memory cell, exact / fast samplers,
# cap plane, strict, steer), sampler, Morton sort + rows, scan + gather, pipelined host path,
# batch driver (commit hash tables, speculative windows, spec_truncate, uint16 wrap), linking,
# attachment, wire formats.  Each tool runs the same pytest selection; the logs and a summary
# land in gpurun_out/<tag>/.
# Usage: bash profiles/sanitize.sh <tag> [tool ...]   (default tools: memcheck racecheck synccheck)
set -u
tag=$1; shift
tools=${*:-memcheck racecheck synccheck}
out=gpurun_out/$tag
mkdir -p "$out"
SEL="tests/test_gpu_parity.py::test_cuda_matches_reference_golden
tests/test_gpu_parity.py::test_cuda_sampler_matches_reference_golden
tests/test_gpu_parity.py::test_every_kernel_variant_bit_exact
tests/test_gpu_parity.py::test_rows_api_equals_csr_and_oracle
tests/test_gpu_parity.py::test_pipelined_host_path_matches
tests/test_gpu_parity.py::test_degenerate_dims_bit_exact
tests/test_driver.py::test_device_driver_matches_reference
tests/test_driver.py::test_device_driver_prefilled_counts_and_uint16_wrap
tests/test_driver.py::test_device_driver_long_segments_global_hash_tables
tests/test_link.py::test_device_link_matches_reference
tests/test_link.py::test_device_grow_matches_reference
tests/test_io.py"
for tool in $tools; do
  timeout 1500 compute-sanitizer --tool "$tool" --target-processes all --print-limit 50 \
    --log-file "$out/sanitize_$tool.log" \
    python -m pytest $SEL -m gpu -q -p no:cacheprovider > "$out/sanitize_${tool}_pytest.log" 2>&1
  rc=$?
  errs=$(grep -h "ERROR SUMMARY" "$out/sanitize_$tool.log" | sort | uniq -c | tr '\n' ';')
  echo "$tool: rc=$rc $(tail -1 "$out/sanitize_${tool}_pytest.log") | $errs"
done
