"""CPU oracle for the RAFEM hot path — TEST INFRASTRUCTURE ONLY (see rafem_oracle.py)."""
