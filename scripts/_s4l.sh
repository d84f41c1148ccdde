for l in lean2 head; do
  echo "=== $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 300 python scripts/vb_sweep.py "vb_debug=0" "dl_buffers=4,vocab_chunk=3072" "dl_buffers=4,vocab_chunk=2560" "dl_buffers=4,vocab_chunk=2048" "dl_buffers=4" "vb_debug=0" 2>&1 | grep -v Warn | cut -c1-130
done
echo "=== trace lean2 nbuf4"; ATTNSM_LIB=$PWD/ablib/lean2.so timeout 120 python scripts/vb_trace.py dl_buffers=4 vocab_chunk=3072 2>&1 | grep "span first\|G1 dl\|G3 dHc\|G2 dW\|MMA-busy"
