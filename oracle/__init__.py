"""Test-only CPU checkers (see oracle/oracle.py and oracle/ref_driver.cpp)."""
