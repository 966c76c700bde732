"""Import-only stand-in for scikit-image (absent; see ../tifffile.py)."""
