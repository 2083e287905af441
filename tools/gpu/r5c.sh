for v in ppf0 ppf ppf0 ppf; do echo "== $v"; python tools/cols_time.py build/variants/$v.so 2>&1 | grep -E "r=(4000|3000|1000|4096) "; done
