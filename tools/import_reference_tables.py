"""Convert the reference's bundled physics data into the package's JSON table file.

Run in the build container (the reference tree does not exist on GPU boxes):

    python tools/import_reference_tables.py [/root/reference/proj/data]

Reads REF's text formats with the package's own parsers (which follow
material.cpp:129-223, spectrum.cpp:32-60, detector_response.cpp:50-79) and writes
paper_2201_13191_b200/data/xscat_tables.json.  Values are stored as
``float.hex`` strings so the round trip is exact.  The Kramers 150 kVp
spectrum of BASELINE config 2 is derived later from these tables
(paper_2201_13191_b200.inputs.kramers_spectrum), not stored.
"""
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2201_13191_b200 import inputs  # noqa: E402


def main():
    data = pathlib.Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/proj/data")
    out = {"source": "reference proj/data (materials, spectra, detector)", "materials": {},
           "spectra": {}, "detector": {}}
    for p in sorted((data / "materials").glob("*.mat")):
        m = inputs.load_material(p)
        out["materials"][m.name] = m.to_json()
    for p in sorted((data / "spectra").glob("*.csv")):
        s = inputs.load_spectrum(p)
        out["spectra"][p.stem] = s.to_json()
    for p in sorted((data / "detector").glob("*.csv")):
        r = inputs.load_detector_response(p)
        out["detector"][p.stem] = r.to_json()
    dst = ROOT / "paper_2201_13191_b200" / "data" / "xscat_tables.json"
    dst.write_text(json.dumps(out, indent=0, sort_keys=True))
    print("wrote", dst)


if __name__ == "__main__":
    main()
