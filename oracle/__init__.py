"""ORACLE — TEST INFRASTRUCTURE ONLY (see pyoracle.py)."""
