export PYTHONPATH=$PWD
python tools/sanitize_driver.py
bash tools/sanitize.sh
