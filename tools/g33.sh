P=tests/test_gpu_parity.py
run() { timeout 900 python -m pytest -q -m gpu "$@" > /tmp/pp.txt 2>&1; echo "$(tail -1 /tmp/pp.txt) :: $*"; }
run tests/test_gpu_large.py::test_L4096_forward_top_orders "$P::test_static_pivot_factorisation_matches_first_call" "$P::test_large_L_inverse_rings_match_oracle"
run tests/test_gpu_large.py::test_L2048_inverse_rings tests/test_gpu_large.py::test_L2048_forward_random_samples "$P::test_static_pivot_factorisation_matches_first_call" "$P::test_large_L_inverse_rings_match_oracle"
run tests/test_gpu_large.py::test_L4096_forward_top_orders "$P::test_large_L_inverse_rings_match_oracle"
run tests/test_gpu_large.py::test_L4096_forward_top_orders "$P::test_static_pivot_factorisation_matches_first_call"  "$P::test_windowed_forward_matches_resident"
