"""Parity oracle for the tilepipe B200 hot path — TEST INFRASTRUCTURE ONLY.

CPU restatements of the reference algorithm (pipeline_ref, resample_ref) and of the
detector placed behind the reference's Detector boundary (yolo_ref). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may use
this package, and only as the checker or the timed CPU reference. The product package
(paper_1810_10551_b200) never imports it.
"""
