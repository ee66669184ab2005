"""CPU checkers for the RASTER path — TEST INFRASTRUCTURE ONLY (see
raster_oracle.h). Importable only by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline/reference leg."""
