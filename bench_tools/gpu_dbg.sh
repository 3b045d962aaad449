make -j8 all > /dev/null 2>&1
timeout 300 compute-sanitizer --print-limit 5 python bench_tools/sanitize_case.py attn_bf16 2>&1 | head -40
