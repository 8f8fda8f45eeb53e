CASES='mfd mfd-escape mfd-escape-coop mfd-ramp' TAG=_mfd_eager TOOLS=racecheck SAN_EAGER=1 bash tools/sanitize.sh
