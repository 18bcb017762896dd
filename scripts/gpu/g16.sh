timeout 900 python -m pytest tests/test_custom_semiring.py tests/test_cpp_facade.py -x -q 2>&1 | tail -15
