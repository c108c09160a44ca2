# sourced by tools/run*.sh: refuse to run GPU work against a library older than its sources
python -c "import sys; sys.path.insert(0,'.'); from paper_2005_09158_b200 import build; sys.exit(1 if build._stale() else 0)" || { echo "STALE libparadiag.so"; exit 3; }
