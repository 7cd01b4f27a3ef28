"""Import stub: scikit-image is absent in this image; the reference's guide.py
imports skimage.feature.canny at module top (guide.py:20).  Only spline
auto-detection uses it, which is outside the fill path."""
