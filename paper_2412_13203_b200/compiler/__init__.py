"""Offline graph compiler: recurrence DAG search (Alg. 1) and CUDA emission."""
