bash tools/ab.sh "m3 m4 m4p0 m5" c2
bash tools/ab.sh "m3 m4 m4p0" c3
