for b in 1 16; do
  echo "== full B=$b"; B=$b python scratch/prof_layer.py
  echo "== no compute B=$b"; RTNQ_WGEMM_DEBUG=1 B=$b python scratch/prof_layer.py
  echo "== no act B=$b"; RTNQ_WGEMM_DEBUG=2 B=$b python scratch/prof_layer.py
  echo "== neither B=$b"; RTNQ_WGEMM_DEBUG=3 B=$b python scratch/prof_layer.py
  echo "== ctas148 B=$b"; RTNQ_WGEMM_CTAS=148 B=$b python scratch/prof_layer.py
done
