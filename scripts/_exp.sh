python scripts/vb_trace.py
python scripts/vb_trace.py vb_debug=1
python scripts/vb_trace.py vb_debug=2
python scripts/vb_trace.py vb_debug=3
python scripts/vb_trace.py vb_debug=7
