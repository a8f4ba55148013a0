python tools/diag_variance2.py bf,torch,bf,bf
python tools/diag_variance2.py torch,bf,bf
python tools/diag_variance2.py bfw1,bf,bfw1
python tools/diag_variance2.py bf,bf,bf keep
